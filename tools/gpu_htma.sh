#!/bin/bash
# TMA spectrum ring (OLSB_HTMA) vs the default TEX path: parity + timings
mkdir -p gpurun_out
L=gpurun_out/htma.log
: > $L
timeout 900 python -m pytest tests/test_gpu_engines.py -q -x -k tma >> $L 2>&1
for v in 0 1 2 3; do
  echo "== OLSB_HTMA=$v" >> $L
  OLSB_HTMA=$v timeout 300 python tools/time_graph.py cfg1 cfg1_f2 cfg4_m8_f1 >> $L 2>&1
  OLSB_HTMA=$v timeout 600 python tools/time_cfg.py cfg3 cfg2_n1024 cfg2_n2048 cfg2_n4096 cfg4_m8_f8 >> $L 2>&1
done
