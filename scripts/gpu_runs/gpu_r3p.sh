mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "minimum_window" 2>&1 | tail -25 | tee gpurun_out/pytest_minwin_r3p.log
