mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -x > gpurun_out/r5d_next.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r5d_tests.log 2>&1
