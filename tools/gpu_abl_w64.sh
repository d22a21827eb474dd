mkdir -p gpurun_out; : > gpurun_out/abl.log
for d in 0 1 5 7; do for v in 1 0; do echo "== OLSB_W64=$v OLSB_DEBUG=$d" >> gpurun_out/abl.log; OLSB_W64=$v OLSB_DEBUG=$d timeout 300 python tools/time_cfg.py cfg3 >> gpurun_out/abl.log 2>&1; done; done
