# new tiny-n parity cases, then the whole GPU suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "tiny_n or fewer_rows" 2>&1 | tail -15 | tee gpurun_out/pytest_tiny_r3o.log
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_r3o.log
