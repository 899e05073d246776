#!/usr/bin/env bash
# K1b kernels A/B (SDMD_K1B = v1 | tma | reg) on the batched push: gpurun -- 'bash scripts/gpu_k1b.sh TAG'
TAG=${1:-k1b}
mkdir -p gpurun_out; export CUDA_DEVICE_MAX_CONNECTIONS=32
for K in reg v1 tma; do
  for C in C4 C3 C2; do
    SDMD_K1B=$K timeout 600 python scripts/bench_batch.py --only $C --modes batch,catchup --frames 200 \
      2>&1 | sed "s/^{/{\"kernel\": \"$K\", /" >> gpurun_out/${TAG}_ab.jsonl
  done
done
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -k "push_batch" > gpurun_out/${TAG}_tests.log 2>&1
