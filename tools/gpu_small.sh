#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/small.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for v in 1 0; do echo "== OLSB_SF_PREF=$v" >> gpurun_out/small.log; OLSB_SF_PREF=$v timeout 300 python tools/time_graph.py cfg1 cfg1_f2 cfg4_m8_f1 cfg4_m32_f1 >> gpurun_out/small.log 2>&1; done
timeout 300 python tools/time_cfg.py cfg3 cfg2_n1024 cfg4_m8_f8 >> gpurun_out/small.log 2>&1
