mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "buildup" 2>&1 | tail -15
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
