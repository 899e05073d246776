mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "device_indices or bad_indices or sparse" 2>&1 | tail -25 | tee gpurun_out/pytest_devidx_r3s.log
