mkdir -p gpurun_out
echo v1; timeout 300 python scripts/k1_micro.py 30 v1 2>&1 | tail -1
echo v2; timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1
for v in l2s1 l2s2 l3s2 dbg1 dbg2 nb16l2; do echo $v; SDMD_LIB=$PWD/variants/libsdmd_$v.so timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1; done
echo v1; timeout 300 python scripts/k1_micro.py 30 v1 2>&1 | tail -1
