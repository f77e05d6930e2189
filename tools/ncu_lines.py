"""Per-CUDA-line warp-stall samples from `ncu --page source --csv --print-source cuda,sass`.

    ncu -i rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows:
    if len(r) <= si or r[0] in ("Line No", "File Path", "Function Name") or r[2] != "-":
        continue          # CUDA-line rows carry '-' in the SASS address column
    try:
        data.append((int(r[si]), int(r[0]), r[1][:100]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for v, ln, src in sorted(data, reverse=True)[:top]:
    print(f"{v:8d} {100 * v / tot:5.1f}%  {ln:5d}  {src}")
