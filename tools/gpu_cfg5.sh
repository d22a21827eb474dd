#!/bin/bash
# cfg5 tests + bench legs: N=1 bench line (with the cfg5 leg) and an
# emulated 2/4/8-rank cfg5 run on one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "cfg5 or halo or shard" > gpurun_out/pytest_cfg5.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
for g in 2 4 8; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-cufft --emulate-ranks $g > gpurun_out/bench_emul$g.json 2> gpurun_out/bench_emul$g.err
done
echo done
