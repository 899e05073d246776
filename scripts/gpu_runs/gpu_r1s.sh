mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
timeout 300 python scripts/diag_k4.py 100 128 200 2>&1 | tee gpurun_out/diag_k4_r1s.jsonl | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['m'], d['cycles'], round(d['k4_ms_avg'],3))"
timeout 900 python scripts/bench_configs.py --workers 20 --out gpurun_out/configs_w20_r1s.md 2>&1 | tail -5
timeout 900 python scripts/bench_configs.py --workers 16 --out gpurun_out/configs_w16_r1s.md 2>&1 | tail -5
