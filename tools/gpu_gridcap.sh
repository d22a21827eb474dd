#!/bin/bash
# small cells: CTAs per SM cap (OLSB_GRID_CAP) -> items per CTA, pipelining
# through the next-item L2 prefetch
mkdir -p gpurun_out
L=gpurun_out/gridcap.log
: > $L
for cap in 0 1 2 3; do
  echo "== OLSB_GRID_CAP=$cap" >> $L
  OLSB_GRID_CAP=$cap timeout 300 python tools/time_graph.py cfg1 cfg1_f2 cfg4_m8_f1 cfg4_m32_f1 cfg4_m8_f8 >> $L 2>&1
done
