mkdir -p gpurun_out
echo v1; timeout 300 python scripts/k1_micro.py 30 v1 2>&1 | tail -2
echo v2; timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -2
for v in nb16 nb8; do echo $v; SDMD_LIB=$PWD/variants/libsdmd_$v.so timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -2; done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 600 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 8 2>&1 | tail -1 | cut -c1-900
