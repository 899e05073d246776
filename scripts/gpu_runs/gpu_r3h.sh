export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "two_ranks_one_gpu_sparse" 2>&1 | tail -15
