#!/bin/bash
# N = 4096 two-warp engine: parity suite, timing vs the E = 16 engine, ncu
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
: > gpurun_out/time_w64x2.log
for v in 1 0; do
  echo "== OLSB_W64X2=$v" >> gpurun_out/time_w64x2.log
  OLSB_W64X2=$v timeout 300 python tools/time_cfg.py cfg2_n4096 cfg5_shard8 >> gpurun_out/time_w64x2.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 1 -c 1 -f -o gpurun_out/prof_w64x2 python tools/prof_cfg.py cfg5_shard8 2 > gpurun_out/prof_w64x2.log 2>&1
ncu -i gpurun_out/prof_w64x2.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_w64x2_src.csv 2>/dev/null
echo done
