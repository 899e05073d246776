# worker split sweep after moving eig(Ã) into K4a (C4, 20 steps x 5 repeats each), with timelines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export CUDA_DEVICE_MAX_CONNECTIONS=32
for cfg in "6 0" "2 4" "3 4" "4 3" "2 3" "4 5"; do
  set -- $cfg
  W=$1; WA=$2
  if [ "$WA" = "0" ]; then unset SDMD_WA; else export SDMD_WA=$WA; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --workers $W --no-cpu-baseline --timeline gpurun_out/r5j_tl_w${W}_a${WA}.npy > gpurun_out/r5j_bench_w${W}_a${WA}.json 2> gpurun_out/r5j_bench_w${W}_a${WA}.err
done
unset SDMD_WA
