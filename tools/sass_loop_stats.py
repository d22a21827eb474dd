"""Static instruction mix of the fused kernel's filter loop (SASS)."""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1910_01972_b200/libolsb.so"
logn = sys.argv[2] if len(sys.argv) > 2 else "11"
prec = sys.argv[3] if len(sys.argv) > 3 else "f"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True,
                      text=True).stdout
key = sys.argv[4] if len(sys.argv) > 4 else f"KCfgI{prec}Li{logn}E"
blk = [b for b in sass.split("Function : ") if "fused_c2c_kernel" in b.split("\n")[0] and key in b.split("\n")[0]][0]
ins = []
for l in blk.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*)", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
# filter loop = from the first LDS.128 after the forward FFT (spectrum read)
# to the backward branch that follows the last STG
stg = [a for a, o, _ in ins if o.startswith("STG")]
last = stg[-1]
back = [(a, rest) for a, o, rest in ins if o == "BRA" and a > last]
tgt = None
for a, rest in back:
    m = re.search(r"0x([0-9a-f]+)", rest)
    if m and int(m.group(1), 16) < last:
        tgt = int(m.group(1), 16)
        end = a
        break
body = [o for a, o, _ in ins if tgt <= a <= end]
c = Counter(o.split(".")[0] for o in body)
fp = sum(c[k] for k in ("FFMA", "FADD", "FMUL", "FFMA2", "FADD2", "FMUL2"))
print(f"loop {hex(tgt)}..{hex(end)}: {len(body)} instr, FP {fp}, non-FP {len(body) - fp}")
print(c.most_common(40))
