#!/usr/bin/env bash
# One `ncu --set full` capture of the dominant kernel (K1 with the fused background, C4) for the
# roofline's `traffic` field: gpurun --timeout 1800 -- 'bash scripts/gpu_ncu_k1.sh TAG'
set -u
TAG=${1:-k1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k1v2_kernel.*bool.1" -s 5 -c 1 -o gpurun_out/${TAG}_k1_full \
  python bench.py --steps 8 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu -i gpurun_out/${TAG}_k1_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_k1_full_raw.csv 2>&1
