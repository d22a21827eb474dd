#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/w32x2.log
OLSB_W32X2=1 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_w32x2.log 2>&1
for v in 1 0; do echo "== OLSB_W32X2=$v" >> gpurun_out/w32x2.log; OLSB_W32X2=$v timeout 300 python tools/time_cfg.py cfg3 cfg2_n2048 >> gpurun_out/w32x2.log 2>&1; done
OLSB_W32X2=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 1 -c 1 -f -o gpurun_out/prof_w32x2 python tools/prof_cfg.py cfg3 2 > gpurun_out/prof_w32x2.log 2>&1
ncu -i gpurun_out/prof_w32x2.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_w32x2_src.csv 2>/dev/null
