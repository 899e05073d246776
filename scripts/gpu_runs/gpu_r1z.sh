mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_r1z.md 2>&1 | tail -6
timeout 300 python scripts/diag_k4.py 100 2>&1 | tail -1 | cut -c1-300
