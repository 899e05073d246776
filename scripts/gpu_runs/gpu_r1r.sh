mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "batch" 2>&1 | tail -3
timeout 600 python scripts/bench_batch.py --frames 400 2>&1 | tee gpurun_out/bench_batch_r1r.jsonl | tail -9
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1b_kernel" -s 6 -c 1 -o gpurun_out/k1b_full_r1r python scripts/bench_batch.py --only C4 --frames 64 > /dev/null 2>&1
timeout 600 python bench.py --steps 400 --no-cpu-baseline --e2e-steps 2 2>/dev/null | cut -c1-300
