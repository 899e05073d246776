mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
DBG_T=6 timeout 300 python scripts/dbg_buildup.py > gpurun_out/r5h_dbg.txt 2>&1
DBG_T=3 timeout 600 compute-sanitizer --tool memcheck python scripts/dbg_buildup.py > gpurun_out/r5h_memcheck.txt 2>&1
timeout 600 python scripts/diag_k4.py 100 200 > gpurun_out/r5h_diag_k4.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r5h_tests.log 2>&1
