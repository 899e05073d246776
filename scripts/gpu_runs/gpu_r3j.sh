export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
