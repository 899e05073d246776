# round 2, session 2: validation at HEAD (tests, smoke, bench, launch list, host CPU model, fp64 peak)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
(lscpu; nproc; free -g) > gpurun_out/r5a_host.txt 2>&1
timeout 120 scripts/ubench/dmma_peak > gpurun_out/r5a_dmma_peak.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r5a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5a_smoke.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r5a_bench20.json 2> gpurun_out/r5a_bench20.err
timeout 600 python bench.py > gpurun_out/r5a_bench_default.json 2> gpurun_out/r5a_bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r5a_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r5a_ncu_bench.log 2>&1
