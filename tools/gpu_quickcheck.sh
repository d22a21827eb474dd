#!/bin/bash
# parity suite + all-config timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/time_cfg.py ${CFGS:-cfg1 cfg3 cfg2_n256 cfg2_n512 cfg2_n1024 cfg2_n2048 cfg2_n4096 cfg4_m8_f8 cfg4_m32_f8 cfg5_shard8} > gpurun_out/time_cfg.log 2>&1
echo done
