mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
B="python bench.py --steps 400 --warmup 5 --no-cpu-baseline --e2e-steps 2"
run() { tag=$1; shift; echo "== $tag"; timeout 300 env "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['frac'], r['k4_ms_avg'], r['k1_wait_ms_avg'], d['clocks']['sm_mhz'])"; }
run l8 $B --lag 8
run l9 $B --lag 9
run l8w7 $B --lag 8 --workers 7
timeout 900 python bench.py 2>gpurun_out/bench_err_r1t.log | tee gpurun_out/bench_r1t.json | cut -c1-200
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tee gpurun_out/bench_ref_r1t.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1|k4|commit|gram_|modes_|k3_" -c 400 --csv --log-file gpurun_out/launches_r1t.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1v2" -s 30 -c 1 -o gpurun_out/k1v2bg_full_r1t python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
ls gpurun_out | grep r1t
