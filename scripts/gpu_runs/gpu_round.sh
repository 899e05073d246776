set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15
timeout 900 python bench.py 2>gpurun_out/bench_err.log | tee gpurun_out/bench_r1a.json
tail -5 gpurun_out/bench_err.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_gram|k4_frame|gram_dmma|gram_reduce|commit|k3_" -c 80 --csv --log-file gpurun_out/launches_r1a.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_bench_stdout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_gram_kernel" -s 4 -c 1 -o gpurun_out/k1_full_r1a python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_stdout.log 2>&1
ls -la gpurun_out
