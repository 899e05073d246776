#!/usr/bin/env bash
# K4a on one CTA (m <= 128) vs the 4-CTA cluster: worker-split sweep with timelines and in-pipeline
# phase cycles, then the GPU tests.   gpurun --timeout 3600 -- 'bash scripts/gpu_k4solo.sh TAG [notests]'
TAG=${1:-s}
mkdir -p gpurun_out; export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python scripts/worker_sweep.py C5 C3 --tl gpurun_out/${TAG}_tl > gpurun_out/${TAG}_sweep.jsonl 2>&1
[ "${2:-}" = notests ] && exit 0
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_tests.log 2>&1
