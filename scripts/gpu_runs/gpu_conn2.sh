mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
run() { echo "== WA=$1 W=$2 L=$3 waves=$4"; SDMD_K1_WAVES=$4 SDMD_WA=$1 timeout 600 python bench.py --steps 100 --no-cpu-baseline --workers $2 --lag $3 --e2e-steps 8 --timeline gpurun_out/tl_$1_$2_$3_$4.npy 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(d['value'], d['e2e']['value'], r['k1_ms_avg'], r['k1_gap_ms_avg'], r['k1_wait_ms_avg'], r['k4_ms_avg'], d['clocks']['sm_mhz'])
    else: print(l.rstrip())
"; python scripts/tl_view.py gpurun_out/tl_$1_$2_$3_$4.npy 0 | tail -4; }
run 2 6 12 8
run 3 6 12 8
run 2 6 12 0
run 2 4 8 8
run 3 8 16 8
run 2 5 12 8
