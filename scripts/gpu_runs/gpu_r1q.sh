mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1b_kernel" -s 6 -c 1 -o gpurun_out/k1b_full_r1q python scripts/bench_batch.py --only C4 --frames 64 > /dev/null 2>&1
ls gpurun_out | grep k1b
