mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python bench.py 2>gpurun_out/bench_err_r3l.log | tee gpurun_out/bench_r3l.json | cut -c1-160
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1|k4|commit|gram_|modes_|k3_" -c 400 --csv --log-file gpurun_out/launches_r3l.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
ls gpurun_out | grep r3l
