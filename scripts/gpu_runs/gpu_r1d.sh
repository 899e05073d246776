set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/host_cpu.txt; nproc >> gpurun_out/host_cpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -25 | tee gpurun_out/pytest_gpu_r1d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 | tee gpurun_out/smoke_r1d.log
timeout 900 python bench.py 2>gpurun_out/bench_err_r1d.log | tee gpurun_out/bench_r1d.json
tail -5 gpurun_out/bench_err_r1d.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench_ref_r1d.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_r1d.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_bench_stdout_r1d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_gram_kernel" -s 6 -c 1 -o gpurun_out/k1_full_r1d python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_stdout_r1d.log 2>&1
ls -la gpurun_out
