mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "gram or video or k1 or c4 or c3 or determinism or nonfinite" 2>&1 | tail -3
B="python bench.py --steps 400 --warmup 5 --no-cpu-baseline --e2e-steps 2"
run() { tag=$1; shift; echo "== $tag"; timeout 300 env "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['frac'], r['k4_ms_avg'], r['k1_wait_ms_avg'], d['clocks']['sm_mhz'])"; }
run skip_l9 $B --lag 9
run noskip_l9 SDMD_LIB=variants/libsdmd_noskip.so $B --lag 9
run skip_l8 $B --lag 8
run noskip_l8 SDMD_LIB=variants/libsdmd_noskip.so $B --lag 8
run skip_l10 $B --lag 10
timeout 300 python scripts/bench_batch.py --only C4 --frames 200 2>&1 | head -1
SDMD_LIB=variants/libsdmd_noskip.so timeout 300 python scripts/bench_batch.py --only C4 --frames 200 2>&1 | head -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1v2" -s 14 -c 1 -o gpurun_out/k1v2bg_full_r1u python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_r1u.log 2>&1
ls gpurun_out | grep r1u
