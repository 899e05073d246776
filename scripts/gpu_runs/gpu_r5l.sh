# Aberth certification rate: cluster version (HEAD) vs the single-CTA K4b version (94ee081)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python scripts/aberth_stats.py 120 6 > gpurun_out/r5l_aberth_head.json 2>&1
