"""Filter-chunk sweep (olsb_set_filter_chunk): items = segments x chunks."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_1910_01972_b200 import _lib  # noqa: E402
from time_cfg import time_cfg  # noqa: E402

for name in sys.argv[1:]:
    for ch in (0, 48, 32, 16, 8):
        _lib.call("olsb_set_filter_chunk", ch)
        t, frac = time_cfg(name)
        print(f"{name} chunk {ch}: {t*1e3:.3f} ms {frac*100:.1f}% HBM", flush=True)
    _lib.call("olsb_set_filter_chunk", 0)
