export CUDA_DEVICE_MAX_CONNECTIONS=32
NCCL_DEBUG=WARN timeout 600 python scripts/two_rank_one_gpu.py 2>&1 | tail -15
