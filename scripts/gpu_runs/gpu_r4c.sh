mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests -m gpu -q -x -k "poison or nonfinite or flow_control or batch or host_input" 2>&1 | tail -30 > gpurun_out/r4c_tests.log
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15 >> gpurun_out/r4c_tests.log
timeout 300 python bench.py --steps 200 --warmup 5 > gpurun_out/r4c_bench.json 2> gpurun_out/r4c_bench.err
