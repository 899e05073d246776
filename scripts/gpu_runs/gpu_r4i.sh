mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4b_kernel" -s 6 -c 1 -o gpurun_out/r4i_k4 python scripts/diag_k4.py 200 > gpurun_out/r4i_ncu.log 2>&1
