# device-side sparse index check: new tests, then the whole GPU suite, then C5
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "device_indices or bad_indices" 2>&1 | tail -25 | tee gpurun_out/pytest_devidx_r3r.log
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_r3r.log
