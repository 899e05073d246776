mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "init_window" 2>&1 | tail -25 | tee gpurun_out/pytest_init_r3u.log
