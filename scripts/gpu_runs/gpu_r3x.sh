mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "maximum_workers" 2>&1 | tail -25 | tee gpurun_out/pytest_maxw_r3x.log
