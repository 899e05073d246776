mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
B="python bench.py --steps 400 --warmup 5 --no-cpu-baseline --e2e-steps 2"
run() { tag=$1; shift; echo "== $tag"; timeout 300 env "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['frac'], r['k4_ms_avg'], r['k1_wait_ms_avg'], d['clocks']['sm_mhz'])"; }
run base              $B
run nodmd  SDMD_BG_NODMD=1 $B
run w4l8   $B --workers 4 --lag 8
run w6l8   $B --workers 6 --lag 8
run w6l10  $B --workers 6 --lag 10
run w6l16  $B --workers 6 --lag 16
run w8l16  $B --workers 8
run w8l12  $B --workers 8 --lag 12
run waves4  SDMD_K1_WAVES=4 $B
run waves16 SDMD_K1_WAVES=16 $B
run waves0  SDMD_K1_WAVES=0 $B
