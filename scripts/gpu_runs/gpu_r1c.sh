set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8 | tee gpurun_out/gpu_tests_r1c.log
timeout 900 python bench.py --steps 100 --no-cpu-baseline 2>&1 | tee gpurun_out/bench_r1c_default.json
for wl in "6 12" "8 12"; do set -- $wl; timeout 900 python bench.py --steps 100 --no-cpu-baseline --workers $1 --lag $2 --e2e-steps 8 2>&1 | tee gpurun_out/bench_w$1l$2.json; done
