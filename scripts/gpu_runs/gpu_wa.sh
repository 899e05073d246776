mkdir -p gpurun_out
run() { echo "== WA=$1 W=$2 L=$3"; SDMD_WA=$1 timeout 600 python bench.py --steps 100 --no-cpu-baseline --workers $2 --lag $3 --e2e-steps 4 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['k1_gap_ms_avg'], r['k1_wait_ms_avg'], r['k4_ms_avg'], d['clocks']['sm_mhz'])
    else: print(l.rstrip())
"; }
run 2 6 8
run 3 6 8
run 3 5 8
run 3 4 8
run 4 4 10
