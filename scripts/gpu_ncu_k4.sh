#!/usr/bin/env bash
# One `ncu --set full` capture of K4a (the 4-CTA cluster at m = 200, video window) and of the
# one-CTA K4a (m = 100): gpurun --timeout 1800 -- 'bash scripts/gpu_ncu_k4.sh TAG'
TAG=${1:-k4}
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
for M in 200 100; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"k4a_kernel" -s 4 -c 1 -o gpurun_out/${TAG}_k4a_m${M} \
    python scripts/diag_k4.py $M > gpurun_out/${TAG}_ncu_k4a_m${M}.log 2>&1
  ncu -i gpurun_out/${TAG}_k4a_m${M}.ncu-rep --page raw --csv > gpurun_out/${TAG}_k4a_m${M}_raw.csv 2>&1
done
