set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -25
timeout 600 python scripts/diag_k4.py 2>&1 | tee gpurun_out/diag_k4.log
timeout 900 python bench.py --steps 100 --no-cpu-baseline 2>&1 | tee gpurun_out/bench_iter.json
