#!/bin/bash
# ncu --set full of the fused kernel on one config (OLSB_VARIANT from env)
# usage: bash tools/gpu_prof.sh <name> <cfg>
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 1 -c 1 -f -o gpurun_out/$1 python tools/prof_cfg.py $2 2 > gpurun_out/$1.log 2>&1
ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_src.csv 2>/dev/null
ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
