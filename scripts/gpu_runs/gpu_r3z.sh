mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "determinism" 2>&1 | tail -25 | tee gpurun_out/pytest_det_r3z.log
