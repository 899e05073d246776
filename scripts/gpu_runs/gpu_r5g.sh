mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
DBG_T=4 timeout 300 python scripts/dbg_buildup.py > gpurun_out/r5g_dbg.txt 2>&1
DBG_T=3 timeout 600 compute-sanitizer --tool memcheck python scripts/dbg_buildup.py > gpurun_out/r5g_memcheck.txt 2>&1
DBG_T=3 timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/dbg_buildup.py > gpurun_out/r5g_racecheck.txt 2>&1
DBG_T=3 timeout 600 compute-sanitizer --tool synccheck python scripts/dbg_buildup.py > gpurun_out/r5g_synccheck.txt 2>&1
