mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
cat > /tmp/c3.py <<'PY'
import sys, json, os
sys.path.insert(0, "scripts"); sys.path.insert(0, ".")
import numpy as np, torch, synth
from bench_configs import dense_run
vs = synth.video_config("C3")
pool = torch.empty((400, vs.n), dtype=torch.float32, device="cuda")
for t in range(400):
    pool[t].copy_(vs.frame(t, device="cuda"))
for lag in [int(a) for a in sys.argv[1:]]:
    r = dense_run("C3", pool, vs.n, 100, "f32", 500, 20, background=True, lag=lag)
    print(lag, r["snapshots_per_s"], r["gram_pass_ms"], r["k4_ms_avg"], flush=True)
PY
timeout 600 python /tmp/c3.py 16 20 24 28 32 40 2>&1 | tail -6
