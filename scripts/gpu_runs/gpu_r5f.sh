mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 300 python scripts/dbg_buildup.py > gpurun_out/r5f_dbg.txt 2>&1
SDMD_ATILDE=v1 timeout 300 python scripts/dbg_buildup.py >> gpurun_out/r5f_dbg.txt 2>&1
timeout 600 python scripts/diag_k4.py 100 200 > gpurun_out/r5f_diag_k4.jsonl 2>&1
SDMD_ATILDE=v1 timeout 600 python scripts/diag_k4.py 100 200 >> gpurun_out/r5f_diag_k4.jsonl 2>&1
