mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "video_background_parity or push_batch_c1 or c1_every" 2>&1 | tail -25 > gpurun_out/racecheck_r2y.txt
tail -10 gpurun_out/racecheck_r2y.txt
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "video_background_parity or c1_every" 2>&1 | tail -25 > gpurun_out/synccheck_r2y.txt
tail -6 gpurun_out/synccheck_r2y.txt
