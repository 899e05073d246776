mkdir -p gpurun_out
timeout 600 python scripts/diag_k4.py 100 200 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 600 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 8 --timeline gpurun_out/tl_k4a.npy 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline'])"
python scripts/tl_view.py gpurun_out/tl_k4a.npy 0 | tail -4
