#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/w64pf.log
OLSB_W64=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "grid or cfg or known" > gpurun_out/pytest_w64.log 2>&1
for d in 0 8; do echo "== OLSB_W64=1 OLSB_DEBUG=$d" >> gpurun_out/w64pf.log; OLSB_W64=1 OLSB_DEBUG=$d timeout 300 python tools/time_cfg.py cfg3 cfg2_n2048 >> gpurun_out/w64pf.log 2>&1; done
echo "== E16" >> gpurun_out/w64pf.log; timeout 300 python tools/time_cfg.py cfg3 cfg2_n2048 >> gpurun_out/w64pf.log 2>&1
