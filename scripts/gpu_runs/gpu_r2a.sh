mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "sparse" 2>&1 | tail -8
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_r2a.md 2>&1 | tail -3
