export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python scripts/bench_two_rank_threads.py 2>&1 | tail -3
