set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_bench_r1c.log 2>&1
tail -2 gpurun_out/ncu_bench_r1c.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_gram_kernel" -s 20 -c 1 -o gpurun_out/k1_bg_full_r1c python bench.py --steps 12 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_k1_r1c.log 2>&1
tail -3 gpurun_out/ncu_k1_r1c.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4a_kernel|k4b_kernel" -s 4 -c 2 -o gpurun_out/k4_full_r1c python bench.py --steps 12 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_k4_r1c.log 2>&1
tail -3 gpurun_out/ncu_k4_r1c.log
