mkdir -p gpurun_out
run() { echo "== W=$1 waves=$2 $3"; SDMD_K1_WAVES=$2 timeout 600 python bench.py --steps 200 --no-cpu-baseline --workers $1 --e2e-steps 48 $3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(d['value'], d['e2e']['value'], r['k1_ms_avg'], r['k1_gap_ms_avg'], r['k1_wait_ms_avg'], r['k4_ms_avg'], d['clocks'], d['config']['k1_grid'], d['config']['lag'])
    else: print(l.rstrip())
"; }
run 6 8
run 6 0
run 6 4
run 6 16
run 4 8
run 8 8
