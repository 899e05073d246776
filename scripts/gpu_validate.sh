#!/usr/bin/env bash
# Round validation on one B200 (run through gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash scripts/gpu_validate.sh TAG'
# Writes gpurun_out/TAG_*: GPU test log, smoke, bench (driver command + default), the ncu launch
# list of a short bench run (our kernels only), K4 phase cycles, every-config table.
set -u
TAG=${1:-val}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
(lscpu; nproc) > gpurun_out/${TAG}_host.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench20.json 2> gpurun_out/${TAG}_bench20.err
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
{ time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_reference.json ; } 2> gpurun_out/${TAG}_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:sdmd -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 20 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 600 python scripts/diag_k4.py 100 128 200 > gpurun_out/${TAG}_diag_k4.jsonl 2>&1
timeout 1800 python scripts/bench_configs.py --frames 500 --workers 20 --out gpurun_out/${TAG}_configs.md \
  > gpurun_out/${TAG}_configs.jsonl 2>&1
timeout 600 python scripts/score_stream.py --config C3 --frames 400 --out gpurun_out/${TAG}_score_c3.json \
  > gpurun_out/${TAG}_score_c3.log 2>&1
