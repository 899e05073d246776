mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"modes_tc_kernel" -s 4 -c 1 -o gpurun_out/k2modes_full_r3b python scripts/k2_bench.py > /dev/null 2>&1
ls gpurun_out | grep r3b
