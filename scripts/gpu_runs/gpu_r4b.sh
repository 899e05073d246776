mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 2>&1 | tail -30 > gpurun_out/r4b_tests.log
