#!/bin/bash
# bench line + reference arm + ncu launch list + full ncu capture (cfg3)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-cufft > gpurun_out/bench_ncu.log 2>&1
bash tools/gpu_prof.sh prof_bench cfg3
echo done
