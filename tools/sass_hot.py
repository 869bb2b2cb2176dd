"""Hot SASS instructions of an ncu report (source page): samples and the top
stall reasons per instruction, in program order, for lines above a threshold.

usage: python tools/sass_hot.py report.ncu-rep [min_samples]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = 0
out = []
for k, r in enumerate(rows[2:]):
    try:
        s = int(r[ix["# Samples"]])
    except (ValueError, IndexError):
        continue
    tot += s
    if s >= thr:
        top = sorted(((int(r[ix[h]]), h[6:]) for h in stalls if r[ix[h]].isdigit() and int(r[ix[h]]) > 0), reverse=True)[:3]
        out.append((k, s, r[ix["Source"]].strip()[:60], top))
for k, s, src, top in out:
    print(f"{k:5d} {s:6d}  {src:60s} {' '.join(f'{n}:{v}' for v, n in top)}")
print("total samples", tot)
