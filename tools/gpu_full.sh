#!/bin/bash
# full GPU check: parity suite, smoke, comparison sweep, per-config timing
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/compare_cufft.py > gpurun_out/compare_cufft.jsonl 2> gpurun_out/compare_cufft.err
timeout 600 python tools/time_cfg.py ${CFGS:-cfg1 cfg3 cfg2_n256 cfg2_n512 cfg2_n1024 cfg2_n2048 cfg2_n4096 cfg4_m8_f8 cfg4_m32_f8} > gpurun_out/time_cfg.log 2>&1
echo done
