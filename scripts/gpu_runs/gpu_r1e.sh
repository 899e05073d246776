mkdir -p gpurun_out
echo micro; timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -2
for w in 4 6 8; do echo workers$w; timeout 600 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 2 --workers $w --timeline gpurun_out/tl_w$w.npy | cut -c1-120; python -c "import json,sys; d=json.load(open('/dev/stdin')); print(d['roofline'])" < /dev/null 2>/dev/null; done
for l in 6 8; do echo lag$l; timeout 600 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 2 --lag $l > gpurun_out/b_lag$l.json; cut -c1-120 gpurun_out/b_lag$l.json; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k4|commit|gram_|modes_|k3_" -c 400 --csv --log-file gpurun_out/launches_r1e.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_bench_stdout_r1e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_gram" -s 20 -c 1 -o gpurun_out/k1bg_full_r1e python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full_stdout_r1e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4" -s 10 -c 2 -o gpurun_out/k4_full_r1e python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_k4_stdout_r1e.log 2>&1
ls gpurun_out
