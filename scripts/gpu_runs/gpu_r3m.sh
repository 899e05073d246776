export CUDA_DEVICE_MAX_CONNECTIONS=32
for lib in "" "SDMD_LIB=variants/libsdmd_small24.so" "SDMD_LIB=variants/libsdmd_small20.so"; do
  echo "== ${lib:-small32}"
  env $lib timeout 300 python scripts/diag_k4.py 100 128 200 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    c=d['cycles']; print(d['m'], 'qr', c['qr'], 'k4b', c['qr']+c['eigvec_c'], 'sweeps', d['ms_sweeps'], 'its', d['qr_block_its'])"
done
