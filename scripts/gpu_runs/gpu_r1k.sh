mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 1200 python scripts/bench_configs.py --out gpurun_out/configs_r1k.md 2>&1 | tail -6
