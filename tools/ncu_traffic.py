"""DRAM traffic per b-pixel of the matching kernels from an ncu --set full
report (dev tool; writes the file bench.py reads for roofline.traffic).

python tools/ncu_traffic.py report.ncu-rep pixels_per_launch out.json
"""
import csv
import io
import json
import subprocess
import sys

rep, px, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
col = {k: h.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
names = {"k_match_refine": "k_match_refine", "k_prep": "k_prep"}
res = {}
for r in rows[2:]:
    kname = r[col["Kernel Name"]]
    key = next((v for k, v in names.items() if k + "(" in kname or kname.endswith(k)), None)
    if key is None or key in res:
        continue
    rd = float(r[col["dram__bytes_read.sum"]]) * scale.get(units[col["dram__bytes_read.sum"]], 1)
    wr = float(r[col["dram__bytes_write.sum"]]) * scale.get(units[col["dram__bytes_write.sum"]], 1)
    res[key] = {"kernel": kname, "dram_bytes_read": rd, "dram_bytes_write": wr,
                "dram_bytes_per_px": (rd + wr) / px, "pixels_in_launch": px,
                "duration_under_ncu": r[col["gpu__time_duration.sum"]] + " " + units[col["gpu__time_duration.sum"]]}
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
