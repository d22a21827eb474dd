#!/bin/bash
# N = 4096 split-coupling exchanges (OLSB_N3) vs the default: parity + timings
mkdir -p gpurun_out
L=gpurun_out/n3.log
: > $L
timeout 600 python -m pytest tests/test_gpu_engines.py -q -x -k N3 >> $L 2>&1
for v in 0 1 0 1; do
  echo "== OLSB_N3=$v" >> $L
  OLSB_N3=$v timeout 300 python tools/time_cfg.py cfg2_n4096 cfg5_shard8 >> $L 2>&1
done
