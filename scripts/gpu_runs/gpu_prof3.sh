set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_gram|k4a_|k4b_|gram_dmma|gram_reduce|ghist|commit_kernel|modes" --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_bench_r1c.log 2>&1
tail -2 gpurun_out/ncu_bench_r1c.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_gram_kernel" -s 8 -c 1 -o gpurun_out/k1_bg_full_r1c python bench.py --steps 12 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_k1_r1c.log 2>&1
tail -3 gpurun_out/ncu_k1_r1c.log
