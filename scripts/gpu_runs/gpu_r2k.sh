mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_r2k.md 2>&1 | tail -8
