# NEXT-3 (Fourier sparse bases, pixel-space IDCT background), NEXT-4 scoring, first-window background
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r5b_next.log
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r5b_tests.log
