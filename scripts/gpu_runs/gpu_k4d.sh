mkdir -p gpurun_out
timeout 300 python scripts/diag_k4.py 100 200 2>&1 | tail -2 | cut -c1-330
SDMD_WARM=0 timeout 300 python scripts/diag_k4.py 200 2>&1 | tail -1 | cut -c1-330
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 8 --timeline gpurun_out/tl_k4d.npy 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['k1_ms_avg'], r['frac'], r['k4_ms_avg'], d['clocks'])"
python scripts/tl_view.py gpurun_out/tl_k4d.npy 0 | tail -4
