#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/pdl.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for v in 1 0; do echo "== OLSB_PDL=$v" >> gpurun_out/pdl.log; OLSB_PDL=$v timeout 300 python tools/time_graph.py cfg1 cfg1_f2 cfg1_f4 cfg4_m8_f1 >> gpurun_out/pdl.log 2>&1; OLSB_PDL=$v timeout 300 python tools/time_cfg.py cfg1 cfg3 >> gpurun_out/pdl.log 2>&1; done
