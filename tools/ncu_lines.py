"""Per-source-line instruction / stall totals from an ncu report (dev tool).

python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kern, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
iE = hdr.index("Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
agg, src, line = {}, {}, None


def num(x):
    try:
        return float(x)
    except ValueError:
        return None


for r in rows:
    if len(r) < len(hdr):
        continue
    if r[0] and num(r[0]) is not None:
        line = int(r[0])
        src[line] = r[1]
    if r[2] and line is not None and num(r[iE]) is not None:
        a = agg.setdefault(line, [0.0, 0.0])
        a[0] += num(r[iE])
        a[1] += num(r[iS]) or 0.0
te = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print(f"total warp-instr {te:.4g}, stall samples {ts:.4g}")
for ln, (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} instr {e / te * 100:5.1f}%  stall {s / ts * 100:5.1f}%  {src.get(ln, '')[:70].strip()}")
