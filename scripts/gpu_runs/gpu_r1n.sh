mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 300 python scripts/diag_k4.py 100 128 200 2>&1 | tee gpurun_out/diag_k4_r1n.jsonl | cut -c1-600
timeout 300 python scripts/k2_bench.py 2>&1 | tee gpurun_out/k2_bench_r1n.jsonl | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gram_tc_kernel" --csv --log-file gpurun_out/k2_launches_r1n.csv python scripts/k2_bench.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k4a_kernel" -s 4 -c 1 -o gpurun_out/k4a_full_r1n python scripts/diag_k4.py 100 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k4b_kernel" -s 4 -c 1 -o gpurun_out/k4b_full_r1n python scripts/diag_k4.py 100 > /dev/null 2>&1
timeout 900 python scripts/bench_configs.py --workers 16 --lag 12 --out gpurun_out/configs_w16_r1n.md 2>&1 | tail -5
ls gpurun_out
