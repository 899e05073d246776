mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1200 python scripts/bench_configs.py 2>&1 | grep '^{' | tee gpurun_out/configs_r3za.jsonl | cut -c1-170
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv | tee -a gpurun_out/configs_r3za.jsonl
