mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 600 python bench.py --steps 400 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['frac'], r['k4_ms_avg'], r['k1_wait_ms_avg'], d['clocks']['sm_mhz'], d['config']['lag'])"
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_r2m_w20.md 2>&1 | tail -8
timeout 900 python scripts/bench_configs.py --workers 22 --out gpurun_out/configs_r2m_w22.md 2>&1 | tail -8
