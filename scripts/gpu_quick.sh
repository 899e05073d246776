#!/usr/bin/env bash
# Quick check: K4 phase cycles, every config, the GPU tests.  gpurun -- 'bash scripts/gpu_quick.sh TAG'
TAG=${1:-q}
mkdir -p gpurun_out; export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 300 python scripts/diag_k4.py 16 100 150 200 > gpurun_out/${TAG}_diag.jsonl 2>&1
timeout 1200 python scripts/bench_configs.py --frames 400 --workers 20 --out gpurun_out/${TAG}_configs.md > gpurun_out/${TAG}_configs.jsonl 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_tests.log 2>&1
