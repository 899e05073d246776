export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python scripts/bench_batch.py --only C1 --frames 400 2>&1 | tail -3
