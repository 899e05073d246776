mkdir -p gpurun_out
timeout 600 python scripts/diag_k4.py 200 2>&1 | tee gpurun_out/diag_k4_r1g.log
