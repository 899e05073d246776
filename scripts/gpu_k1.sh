set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 600 python scripts/diag_k4.py 100 150 200 2>&1 | tee gpurun_out/diag_k4.log
timeout 900 python bench.py --steps 100 --no-cpu-baseline --workers 4 2>&1 | tee gpurun_out/bench_iter.json
timeout 900 python bench.py --steps 100 --no-cpu-baseline --workers 8 2>&1 | tee gpurun_out/bench_iter_w8.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 2>&1 | tee gpurun_out/bench_ref.json
