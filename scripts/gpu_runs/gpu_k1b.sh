mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 600 python scripts/k1_micro.py 30 ldg 2>&1 | tee gpurun_out/k1_micro.log
timeout 600 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 48 2>&1 | tee gpurun_out/bench_k1b.json | cut -c1-250
