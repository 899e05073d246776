mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"modes_tc_kernel|gram_tc_kernel" -s 8 -c 2 -o gpurun_out/k2_full_r3a python scripts/k2_bench.py > /dev/null 2>&1
ls gpurun_out | grep r3a
