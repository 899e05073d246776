mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k4a_kernel" -s 4 -c 1 -o gpurun_out/k4a150_full_r3d python scripts/diag_k4.py 150 > /dev/null 2>&1
ls gpurun_out | grep r3d
