#!/bin/bash
# round-end evidence: bench line, reference arm, numba reference timing,
# ncu launch list of the bench, full ncu capture of the cfg3 kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
PYTHONPATH=baseline/_ref timeout 900 python tools/time_numba_ref.py --repeats 2 > gpurun_out/numba_ref.json 2> gpurun_out/numba_ref.err
nproc > gpurun_out/nproc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-cufft --no-cfg5 > gpurun_out/bench_ncu.log 2>&1
bash tools/gpu_prof.sh prof_cfg3 cfg3
echo done
