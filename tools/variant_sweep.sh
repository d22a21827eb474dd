#!/bin/bash
# sweep OLSB_VARIANT over the fused fp32 policies (N = 2048 / 4096)
for v in ${VARIANTS:-0 1 2 3 4 5 6 7}; do
  OLSB_VARIANT=$v timeout 300 python tools/time_cfg.py ${CFGS:-cfg3 cfg2_n4096 cfg2_n2048}
done
