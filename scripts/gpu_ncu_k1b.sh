#!/usr/bin/env bash
# One `ncu --set full` capture of the batched Gram pass K1b (cp.async kernel, C4, k = 8):
#   gpurun --timeout 1800 -- 'bash scripts/gpu_ncu_k1b.sh TAG'
TAG=${1:-k1b}
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
SDMD_K1B=v1 timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k1b_kernel" -s 3 -c 1 -o gpurun_out/${TAG}_k1b_full \
  python scripts/bench_batch.py --only C4 --modes catchup --frames 48 > gpurun_out/${TAG}_ncu_k1b.log 2>&1
ncu -i gpurun_out/${TAG}_k1b_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_k1b_full_raw.csv 2>&1
ncu -i gpurun_out/${TAG}_k1b_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_k1b_source.csv 2>&1
