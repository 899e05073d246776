mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
run() { echo "== WAVES=$1 WA=$2 W=$3 L=$4"; SDMD_K1_WAVES=$1 SDMD_WA=$2 timeout 600 python bench.py --steps 100 --no-cpu-baseline --workers $3 --lag $4 --e2e-steps 4 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['k1_gap_ms_avg'], r['k1_wait_ms_avg'], r['k4_ms_avg'], d['clocks']['sm_mhz'])
    else: print(l.rstrip())
"; }
run 0 2 6 8
run 4 2 6 8
run 8 2 6 8
run 16 2 6 8
run 8 3 6 8
run 8 2 4 8
run 8 2 6 6
