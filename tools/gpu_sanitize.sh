#!/bin/bash
# compute-sanitizer memcheck / racecheck over tools/sanitize_cells.py with the
# default engine and each experimental engine switch (round 2)
mkdir -p gpurun_out
L=gpurun_out/sanitize.log
: > $L
CS=/usr/local/cuda/bin/compute-sanitizer
echo "## plain run" >> $L
timeout 600 python tools/sanitize_cells.py >> $L 2>&1 || echo "plain rc=$?" >> $L
for env in "" "OLSB_W64=1" "OLSB_W64X2=1" "OLSB_W32X2=1" "OLSB_HTMA=1" "OLSB_HTMA=3"; do
  for tool in memcheck racecheck; do
    echo "## $tool ${env:-default}" >> $L
    env $env timeout 1500 $CS --tool $tool --print-limit 20 python tools/sanitize_cells.py 2>&1 \
      | grep -v "^========= COMPUTE-SANITIZER" | tail -12 >> $L
  done
done
