mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "every_frame or c1_every or c2_wake or push_batch" 2>&1 | tail -6
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_r2h.md 2>&1 | tail -8
