mkdir -p gpurun_out
for c in 8 32; do
for wa in 2 3; do
echo "== CONN=$c WA=$wa"
CUDA_DEVICE_MAX_CONNECTIONS=$c SDMD_WA=$wa timeout 600 python bench.py --steps 60 --no-cpu-baseline --e2e-steps 2 --timeline gpurun_out/tl_c${c}_a${wa}.npy | cut -c1-120
python scripts/tl_view.py gpurun_out/tl_c${c}_a${wa}.npy 0 | tail -4
done; done
