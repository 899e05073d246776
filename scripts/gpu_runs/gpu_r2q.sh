mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
B="python bench.py --steps 400 --warmup 5 --no-cpu-baseline --e2e-steps 2"
run() { tag=$1; shift; echo "== $tag"; timeout 300 env "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['frac'], r['k4_ms_avg'], r['k1_wait_ms_avg'], d['clocks']['sm_mhz'])"; }
run pf0 $B
run pf1 SDMD_LIB=variants/libsdmd_pf1.so $B
run pf2 SDMD_LIB=variants/libsdmd_pf2.so $B
run pf4 SDMD_LIB=variants/libsdmd_pf4.so $B
run pf0b $B
run pf2b SDMD_LIB=variants/libsdmd_pf2.so $B
