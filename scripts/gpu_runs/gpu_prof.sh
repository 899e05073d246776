set -x
mkdir -p gpurun_out
./scripts/ubench/fp64_lat | tee gpurun_out/fp64_lat.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k4_frame_kernel" -s 0 -c 1 -o gpurun_out/k4_full python scripts/diag_k4.py 200 > gpurun_out/ncu_k4.log 2>&1
tail -2 gpurun_out/ncu_k4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_gram_kernel" -s 209 -c 1 -o gpurun_out/k1_nobg_full python scripts/k1_micro.py 3 ldg > gpurun_out/ncu_k1a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_gram_kernel" -s 418 -c 1 -o gpurun_out/k1_bg_full python scripts/k1_micro.py 3 ldg > gpurun_out/ncu_k1b.log 2>&1
tail -2 gpurun_out/ncu_k1b.log
