mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>gpurun_out/bench_err_r1l.log | tee gpurun_out/bench_r1l.json | cut -c1-400
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_r1l.md 2>&1 | tail -8
