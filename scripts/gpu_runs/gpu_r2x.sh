mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
export PYTHONUNBUFFERED=1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "c1_every or video_background_parity or sparse_dct or push_batch_c1 or buildup_dmd_every_window" 2>&1 | tail -30 > gpurun_out/memcheck_r2x.txt
tail -8 gpurun_out/memcheck_r2x.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "video_background_parity and 2" 2>&1 | tail -30 > gpurun_out/racecheck_r2x.txt
tail -8 gpurun_out/racecheck_r2x.txt
