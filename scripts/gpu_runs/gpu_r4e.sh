mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x -k "two_ranks or nccl or singular" 2>&1 | tail -60 > gpurun_out/r4e_tests.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 >> gpurun_out/r4e_tests.log
