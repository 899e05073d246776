"""Per-source-line hot spots from `ncu -i REP --page source --csv --print-source cuda,sass -k K`.
Usage: python scripts/ncu_lines.py mix.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = next(r for r in rows if r and r[0] == "Line No")
si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_")]
lines = []
for r in rows:
    if r and r[0] not in ("", "Line No") and r[0].isdigit() and len(r) > ii:
        try:
            s, n = int(r[si]), int(r[ii])
        except ValueError:
            continue
        st = sorted(((int(r[i]) if r[i].isdigit() else 0, c[6:]) for i, c in stall_cols), reverse=True)[:3]
        lines.append((s, n, int(r[0]), r[1][:90], st))
tot = sum(l[0] for l in lines)
print(f"total samples {tot}")
for s, n, ln, src, st in sorted(lines, reverse=True)[:top]:
    print(f"{s:6d} {s/tot:6.1%} inst {n:10d}  L{ln:<5d} {src}  {st}")
