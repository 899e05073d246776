# final validation at the session HEAD: GPU parity suite, smoke, headline bench
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_r3w.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2 | tee gpurun_out/smoke_r3w.log
timeout 900 python bench.py 2>gpurun_out/bench_err_r3w.log | tee gpurun_out/bench_r3w.json | cut -c1-200
