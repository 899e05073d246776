timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -2
for d in 1 2 3; do echo "dbg=$d"; SDMD_K1_DBG=$d timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1; done
timeout 600 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 48 2>&1 | tee gpurun_out/bench_k1c.json | cut -c1-150
