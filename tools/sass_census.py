"""Per-kernel SASS census of the built library: counts of the instructions that
prove which hardware path a kernel uses (tcgen05 MMAs UTC*MMA, TMEM loads
LDTM, TMA bulk copies UBLKCP / tensor TMA UTMALDG / UTMASTG, DMMA, FFMA2 ...).
usage: python tools/sass_census.py [lib.so] > profiles/r02/sass_census.json"""
import json
import re
import subprocess
import sys
from collections import Counter, defaultdict

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2409_08970_b200/lib/libdctplus_b200.so"
OPS = ["UTCHMMA", "UTCIMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "UTMASTG", "DMMA", "HMMA",
       "DFMA", "FFMA2", "FFMA", "SYNCS", "LDGSTS", "MUFU"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
counts = defaultdict(Counter)
name = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        continue
    if name is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(1)
        for o in OPS:
            if op == o or op.startswith(o + "."):
                counts[name][o] += 1


def short(n):
    d = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"dctp::dev::\(anonymous namespace\)::", "", d)
    return d[:160]


out = {short(k): dict(v) for k, v in sorted(counts.items()) if v}
print(json.dumps(out, indent=1))
