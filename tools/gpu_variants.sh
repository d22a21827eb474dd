#!/bin/bash
# GPU parity suite + fused-kernel policy sweep (OLSB_VARIANT) on the cfgs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
for v in ${VARIANTS:-0 1 2 3 4 5 6 7}; do
  OLSB_VARIANT=$v timeout 300 python tools/time_cfg.py ${CFGS:-cfg3 cfg2_n2048 cfg2_n4096} >> gpurun_out/variants.log 2>&1
done
echo done
