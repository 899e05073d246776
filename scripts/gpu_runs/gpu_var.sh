timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
echo base; timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1
for v in ring cb5 cb3 cb6; do echo $v; SDMD_LIB=$PWD/variants/libsdmd_$v.so timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1; done
for c in 50 100; do echo carve$c; SDMD_K1_CARVEOUT=$c timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1; done
echo base; timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1
timeout 600 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 48 2>&1 | tee gpurun_out/bench_k1d.json | cut -c1-150
