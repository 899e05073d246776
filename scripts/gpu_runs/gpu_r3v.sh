mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -x -q -m gpu -k "device_indices_checked or fully_dense_frames or empty_sparse or init_window_nonfinite" > gpurun_out/sanitizer_r3v.log 2>&1
tail -8 gpurun_out/sanitizer_r3v.log
