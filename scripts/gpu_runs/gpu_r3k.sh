mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
for lib in "" "SDMD_LIB=variants/libsdmd_noflags.so"; do
  echo "== ${lib:-flags}"
  env $lib timeout 300 python scripts/diag_k4.py 100 150 200 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['m'], d['sweeps'], 'jacobi', d['cycles']['jacobi'], 'k4ms', round(d['k4_ms_avg'],3))"
  env $lib timeout 600 python scripts/bench_configs.py --out /tmp/x.md 2>&1 | head -3 | tail -2 | cut -c1-140
done
