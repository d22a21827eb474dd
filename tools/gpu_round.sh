#!/bin/bash
# One gpurun call: GPU parity suite, per-config timing, bench line, ncu
# launch list and a full ncu capture of the fused kernel (cfg3).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/time_cfg.py ${CFGS:-cfg1 cfg3 cfg2_n256 cfg2_n512 cfg2_n1024 cfg2_n2048 cfg2_n4096 cfg4_m8_f8 cfg4_m32_f8} > gpurun_out/time_cfg.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_c2c -s 1 -c 1 -o gpurun_out/prof_cfg3 -f python tools/prof_cfg.py cfg3 2 > gpurun_out/ncu_full.log 2>&1
echo done
