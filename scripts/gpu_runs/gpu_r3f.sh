mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>gpurun_out/bench_err_r3f.log | tee gpurun_out/bench_r3f.json | cut -c1-160
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_r3f.md 2>&1 | tail -8
