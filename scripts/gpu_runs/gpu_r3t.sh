mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python scripts/bench_configs.py 2>&1 | grep '"C5' | tee gpurun_out/configs_r3t.jsonl | cut -c1-220
