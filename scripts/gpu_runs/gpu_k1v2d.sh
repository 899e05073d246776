mkdir -p gpurun_out
echo v2; timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1
for v in n16l4 n16l6 l8s2 n16l3 n16l4s4; do echo $v; SDMD_LIB=$PWD/variants/libsdmd_$v.so timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1; done
for v in n16l4 n16l6; do echo bench $v; SDMD_LIB=$PWD/variants/libsdmd_$v.so timeout 600 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 8 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['k1_ms_avg'], d['roofline']['frac'])"; done
