#!/usr/bin/env bash
# Cholesky-preconditioned Jacobi start (SDMD_K4_CHOL=1) vs the S·Q0 start: K4 phase cycles, every
# config, the GPU tests with it on.   gpurun -- 'bash scripts/gpu_k4chol.sh TAG [notests]'
TAG=${1:-ch}
mkdir -p gpurun_out; export CUDA_DEVICE_MAX_CONNECTIONS=32
SDMD_K4_CHOL=1 timeout 300 python scripts/diag_k4.py 16 100 128 150 200 > gpurun_out/${TAG}_diag_chol.jsonl 2>&1
SDMD_K4_CHOL=0 timeout 300 python scripts/diag_k4.py 16 100 128 150 200 > gpurun_out/${TAG}_diag_base.jsonl 2>&1
SDMD_K4_CHOL=1 timeout 1200 python scripts/bench_configs.py --frames 400 --workers 20 --out gpurun_out/${TAG}_configs_chol.md > gpurun_out/${TAG}_configs_chol.jsonl 2>&1
[ "${2:-}" = notests ] && exit 0
SDMD_K4_CHOL=1 timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_tests_chol.log 2>&1
