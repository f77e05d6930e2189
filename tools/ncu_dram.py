"""DRAM bytes per launch of the kernels in an `ncu --set full` report (the
bench line's roofline.traffic):
    python tools/ncu_dram.py rep.ncu-rep workload "command" > profiles/r2/exploit_ncu.json"""
import csv
import io
import json
import subprocess
import sys

rep, workload, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
ri, wi = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
ki, di = hdr.index("Kernel Name"), hdr.index("gpu__time_duration.sum")
units = rows[1]


def val(r, i):
    x = float(r[i].replace(",", ""))
    u = units[i]
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "nsecond": 1,
                "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(u, 1)


each, names, dur = [], [], []
for r in rows[2:]:
    if len(r) == len(hdr):
        each.append(int(val(r, ri) + val(r, wi)))
        dur.append(val(r, di))
        names.append(r[ki][:60])
print(json.dumps({"workload": workload, "kernel": names[0] if names else None,
                  "launches_captured": len(each),
                  "dram_bytes_per_launch": int(sum(each) / max(1, len(each))),
                  "dram_bytes_each": each, "duration_ns_each": [round(x) for x in dur],
                  "source": cmd}, indent=1))
