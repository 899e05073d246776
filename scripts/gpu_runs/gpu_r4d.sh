mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -k "nonfinite or flow_control or sparse_device or singular" 2>&1 | tail -150 > gpurun_out/r4d_tests.log
