mkdir -p gpurun_out
timeout 600 python scripts/diag_k4.py 100 200 2>&1 | tee gpurun_out/diag_k4_r1f.log
echo tma; timeout 300 python scripts/k1_micro.py 30 tma 2>&1 | tail -2
