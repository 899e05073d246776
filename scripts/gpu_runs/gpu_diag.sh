set -x
mkdir -p gpurun_out
timeout 600 python scripts/diag_k4.py 2>&1 | tee gpurun_out/diag_k4.log
timeout 900 python bench.py --steps 100 --no-cpu-baseline 2>&1 | tee gpurun_out/bench_r1b.json
