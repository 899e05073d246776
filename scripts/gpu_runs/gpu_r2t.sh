mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 300 python scripts/diag_k4.py 128 200 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['m'], 'qr', d['cycles']['qr'], 'sweeps', d['ms_sweeps'], 'k4ms', round(d['k4_ms_avg'],3))"
timeout 600 python bench.py --steps 400 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['frac'], r['k4_ms_avg'], r['k1_wait_ms_avg'], d['clocks']['sm_mhz'])"
