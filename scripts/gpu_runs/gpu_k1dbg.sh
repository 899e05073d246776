for d in 0 1 2 3; do echo "dbg=$d"; SDMD_K1_DBG=$d timeout 300 python scripts/k1_micro.py 30 ldg 2>&1 | tail -1; done
