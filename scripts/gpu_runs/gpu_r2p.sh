mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>gpurun_out/bench_err_r2p.log | tee gpurun_out/bench_r2p.json | cut -c1-200
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tee gpurun_out/bench_ref_r2p.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1|k4|commit|gram_|modes_|k3_" -c 400 --csv --log-file gpurun_out/launches_r2p.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1v2" -s 14 -c 1 -o gpurun_out/k1v2bg_full_r2p python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
ls gpurun_out | grep r2p
