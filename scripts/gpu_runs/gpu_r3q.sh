mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "fully_dense_frames" 2>&1 | tail -25 | tee gpurun_out/pytest_sparse_edge_r3q.log
