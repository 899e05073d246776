mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
B="python bench.py --steps 400 --warmup 5 --no-cpu-baseline --e2e-steps 2"
run() { tag=$1; shift; echo "== $tag"; timeout 300 env "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['frac'], r['k4_ms_avg'], r['k1_wait_ms_avg'], d['clocks']['sm_mhz'], d['clocks']['power_w_max'])"; }
run base $B
run h2000 SDMD_LIB=variants/libsdmd_hint2000.so $B
run h20000 SDMD_LIB=variants/libsdmd_hint20000.so $B
run base2 $B
run h2000b SDMD_LIB=variants/libsdmd_hint2000.so $B
SDMD_LIB=variants/libsdmd_hint2000.so timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "video or c4 or c3 or k1_v2" 2>&1 | tail -2
