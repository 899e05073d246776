mkdir -p gpurun_out
SDMD_WA=3 SDMD_K1_WAVES=8 timeout 600 python bench.py --steps 60 --no-cpu-baseline --e2e-steps 2 --timeline gpurun_out/tl_a3w8.npy | cut -c1-200
SDMD_WA=3 SDMD_K1_WAVES=0 timeout 600 python bench.py --steps 60 --no-cpu-baseline --e2e-steps 2 --timeline gpurun_out/tl_a3w0.npy | cut -c1-200
SDMD_WA=4 SDMD_K1_WAVES=8 timeout 600 python bench.py --steps 60 --no-cpu-baseline --e2e-steps 2 --lag 10 --timeline gpurun_out/tl_a4w8.npy | cut -c1-200
