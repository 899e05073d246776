mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -k "c5_scale or c4s_bench" 2>&1 | tail -40 > gpurun_out/r4f_tests.log
timeout 600 python scripts/diag_k4.py 100 128 200 > gpurun_out/r4f_diag_k4.jsonl 2>&1
