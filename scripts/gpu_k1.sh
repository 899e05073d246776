set -x
mkdir -p gpurun_out
timeout 600 python scripts/k1_micro.py 30 ldg,tma 2>&1 | tee gpurun_out/k1_micro.log
timeout 600 python scripts/diag_k4.py 100 200 2>&1 | tee gpurun_out/diag_k4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_gram_kernel" -s 215 -c 1 -o gpurun_out/k1_ldg_bg_full python scripts/k1_micro.py 3 ldg > gpurun_out/ncu_ldg.log 2>&1
tail -3 gpurun_out/ncu_ldg.log
timeout 900 python bench.py --steps 100 --no-cpu-baseline 2>&1 | tee gpurun_out/bench_iter.json
