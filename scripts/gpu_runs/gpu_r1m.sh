mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "modes_tensor or init_window" 2>&1 | tail -4
timeout 300 python scripts/k2_bench.py 2>&1 | tee gpurun_out/k2_bench_v2.jsonl | tail -3
SDMD_K2=v1 timeout 300 python scripts/k2_bench.py 2>&1 | tee gpurun_out/k2_bench_v1.jsonl | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none -k regex:"gram_|modes_" --csv --log-file gpurun_out/k2_launches_r1m.csv python scripts/k2_bench.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gram_tc_kernel|modes_tc_kernel" -s 8 -c 2 -o gpurun_out/k2_full_r1m python scripts/k2_bench.py > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
timeout 900 python scripts/bench_configs.py --workers 16 --out gpurun_out/configs_w16_r1m.md 2>&1 | tail -5
ls gpurun_out
