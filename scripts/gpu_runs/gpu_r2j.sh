mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
cat > /tmp/c2.py <<'PY'
import sys, json, os
sys.path.insert(0, "scripts"); sys.path.insert(0, ".")
import numpy as np, torch, synth
from bench_configs import dense_run
cw = synth.cylinder_wake(); Xc = cw.frames(0, 300)
Xcd = torch.from_numpy(np.ascontiguousarray(Xc.T)).cuda()
W = int(sys.argv[1])
r = dense_run("C2", Xcd, cw.n, 150, "f64", 500, W, r_max=21)
print(W, os.environ.get("SDMD_WA"), r["snapshots_per_s"], r["k4_ms_avg"])
PY
for cfg in "20 10" "10 20" "8 22" "14 16" "6 24"; do set -- $cfg; SDMD_WA=$2 timeout 300 python /tmp/c2.py $1 2>&1 | tail -1; done
