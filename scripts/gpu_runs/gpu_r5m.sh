# Aberth stagnation freeze: failure rate, tests, bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python scripts/aberth_stats.py 120 6 > gpurun_out/r5m_aberth.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r5m_tests.log 2>&1
for W in 6 4; do
timeout 600 python bench.py --steps 20 --warmup 5 --workers $W --no-cpu-baseline --timeline gpurun_out/r5m_tl_w$W.npy > gpurun_out/r5m_bench_w$W.json 2> gpurun_out/r5m_bench_w$W.err
done
