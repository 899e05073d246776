mkdir -p gpurun_out
timeout 300 python scripts/diag_k4.py 200 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 48 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'], d['roofline'])"
