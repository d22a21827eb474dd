#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "cufft or r2r_spectra or real_path or variants" > gpurun_out/pytest_cufft.log 2>&1
: > gpurun_out/cufft_chunks.log
for xc in 16 64 256; do for yc in 32 256 1024; do
  echo "== XCHUNK ${xc}MiB YCHUNK ${yc}MiB" >> gpurun_out/cufft_chunks.log
  OLSB_CUFFT_XCHUNK=$((xc<<20)) OLSB_CUFFT_YCHUNK=$((yc<<20)) timeout 300 python tools/compare_cufft.py cfg3 cfg2_n1024 >> gpurun_out/cufft_chunks.log 2>&1
done; done
echo done
