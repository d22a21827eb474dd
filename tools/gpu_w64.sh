#!/bin/bash
# W64 engine check: parity suite, timing of the store variants vs the E = 16
# engine, ncu capture of the default
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
: > gpurun_out/time_w64.log
for v in ${W64_VARIANTS:-1 2 0}; do
  echo "== OLSB_W64=$v" >> gpurun_out/time_w64.log
  OLSB_W64=$v timeout 300 python tools/time_cfg.py ${CFGS:-cfg3 cfg2_n2048} >> gpurun_out/time_w64.log 2>&1
done
[ -n "$NO_PROF" ] || bash tools/gpu_prof.sh prof_w64 cfg3
