mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r4a_tests.log
timeout 300 python bench.py > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err
nproc > gpurun_out/r4a_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/r4a_host.txt
