mkdir -p gpurun_out
# k1_micro: 208 + 30 no-BG launches, then 208 (no BG during fill) + 30 BG; capture one BG launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_gram_kernel" -s 470 -c 1 -o gpurun_out/k1_bg_bulk python scripts/k1_micro.py 30 ldg > gpurun_out/ncu_k1bulk.log 2>&1
tail -3 gpurun_out/ncu_k1bulk.log
