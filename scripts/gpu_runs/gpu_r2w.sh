mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python bench.py 2>gpurun_out/bench_err_r2w.log | tee gpurun_out/bench_r2w.json | cut -c1-200
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tee gpurun_out/bench_ref_r2w.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1|k4|commit|gram_|modes_|k3_" -c 400 --csv --log-file gpurun_out/launches_r2w.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1v2" -s 14 -c 1 -o gpurun_out/k1v2bg_full_r2w python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
timeout 600 python scripts/bench_batch.py --only C4 --frames 400 2>&1 | tee gpurun_out/bench_batch_r2w.jsonl | tail -3
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_r2w.md 2>&1 | tail -8
ls gpurun_out | grep r2w
