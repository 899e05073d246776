timeout 300 python scripts/h2d_bw.py 2>&1 | tail -4
nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" | head -12
