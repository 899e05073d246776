set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 600 python scripts/k1_micro.py 30 ldg 2>&1 | tee gpurun_out/k1_micro.log
timeout 600 python scripts/diag_k4.py 100 200 2>&1 | tee gpurun_out/diag_k4.log
for wl in "6 8" "8 10" "4 8"; do set -- $wl; timeout 900 python bench.py --steps 100 --no-cpu-baseline --workers $1 --lag $2 --e2e-steps 48 2>&1 | tee gpurun_out/bench_w$1l$2.json; done
