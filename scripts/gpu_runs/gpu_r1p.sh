mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -6
timeout 600 python scripts/bench_batch.py --frames 400 2>&1 | tee gpurun_out/bench_batch_r1p.jsonl | tail -12
B="python bench.py --steps 400 --warmup 5 --no-cpu-baseline --e2e-steps 2"
run() { tag=$1; shift; echo "== $tag"; timeout 300 env "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['frac'], r['k4_ms_avg'], r['k1_wait_ms_avg'], d['clocks']['sm_mhz'])"; }
run w0l8   SDMD_K1_WAVES=0 $B --lag 8
run w0l9   SDMD_K1_WAVES=0 $B --lag 9
run w0l10  SDMD_K1_WAVES=0 $B --lag 10
run w8l9   $B --lag 9
run w0l9w7 SDMD_K1_WAVES=0 $B --lag 9 --workers 7
