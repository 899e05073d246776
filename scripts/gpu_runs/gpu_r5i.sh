# eig(Ã) on the K4a cluster (Aberth over 4 CTAs, QR fallback on CTA 0): diag, tests, bench, launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python scripts/diag_k4.py 100 128 200 > gpurun_out/r5i_diag_k4.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r5i_tests.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r5i_bench20.json 2> gpurun_out/r5i_bench20.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:sdmd -c 400 --csv --log-file gpurun_out/r5i_launches.csv python bench.py --steps 20 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/r5i_ncu_bench.log 2>&1
