# K4a tiled Ã stage + parallel Aberth pairing: diag cycles, full GPU suite, bench (20 steps, repeats)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python scripts/diag_k4.py 100 128 200 > gpurun_out/r5e_diag_k4.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r5e_tests.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r5e_bench20.json 2> gpurun_out/r5e_bench20.err
