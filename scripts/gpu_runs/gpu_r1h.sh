mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 python bench.py 2>gpurun_out/bench_err_r1h.log | tee gpurun_out/bench_r1h.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1|k4|commit|gram_|modes_|k3_" -c 400 --csv --log-file gpurun_out/launches_r1h.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1v2" -s 30 -c 1 -o gpurun_out/k1v2bg_full_r1h python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_dmma" -c 1 -o gpurun_out/k2_full_r1h python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
ls gpurun_out | tail -5
