set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 600 python scripts/k1_micro.py 30 ldg 2>&1 | tee gpurun_out/k1_micro.log
timeout 600 python scripts/diag_k4.py 100 150 200 2>&1 | tee gpurun_out/diag_k4.log
timeout 900 python bench.py --steps 100 --no-cpu-baseline 2>&1 | tee gpurun_out/bench_iter.json
timeout 900 python bench.py --steps 100 --no-cpu-baseline --workers 8 --e2e-steps 4 2>&1 | tee gpurun_out/bench_iter_w8.json
