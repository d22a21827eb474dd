"""Registers / stack of the fused-kernel instantiations in libolsb.so
(cuobjdump -res-usage), keyed by their KCfg arguments and mode."""
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_1910_01972_b200/libolsb.so"
pat = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-res-usage", so], capture_output=True,
                     text=True).stdout.splitlines()
name = None
for line in out:
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    if name and "REG:" in line:
        r = re.search(r"REG:(\d+) STACK:(\d+)", line)
        k = re.search(r"fused_c2c_kernelINS_4KCfgI([fd])((?:Li\d+E)+)EELi(\d)ELb(\d)", name)
        if k:
            args = ",".join(re.findall(r"Li(\d+)E", k.group(2)))
            label = f"{k.group(1)}<{args}> mode {k.group(3)} xr {k.group(4)}"
            if pat in label:
                print(f"{label:48s} REG {r.group(1):>4} STACK {r.group(2)}")
        name = None
