"""Record one kernel's dram traffic (read + write bytes of one launch) from an ncu --set full raw
CSV export into profiles/traffic.json, tagged with the kernel-source hash bench.py checks.
Usage: python scripts/ncu_traffic.py <raw.csv> <workload> <label> [capture-name]"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import csrc_hash  # noqa: E402

raw, workload, label = sys.argv[1:4]
cap = sys.argv[4] if len(sys.argv) > 4 else os.path.basename(raw)
rows = list(csv.reader(open(raw)))
hdr, units = rows[0], rows[1]
d = dict(zip(hdr, rows[2]))
u = dict(zip(hdr, units))


def nbytes(k):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[k]]
    return float(d[k].replace(",", "")) * scale


tot = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    "traffic.json")
t = json.load(open(path)) if os.path.exists(path) else {}
t.setdefault(workload, {})[label] = {
    "dram_bytes": int(tot), "kernel": d.get("Kernel Name", "")[:120],
    "duration": d.get("gpu__time_duration.sum"), "csrc_hash": csrc_hash(), "capture": cap}
json.dump(t, open(path, "w"), indent=1, sort_keys=True)
print(workload, label, int(tot))
