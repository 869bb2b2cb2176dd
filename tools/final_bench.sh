#!/bin/bash
# End-of-round bench set (GPU box): every config through bench.py, the
# reference arm, written to gpurun_out/final/.
set -u
out=gpurun_out/final
mkdir -p $out
python bench.py > $out/bench_final.json 2> $out/bench_final.err
python bench.py --impl reference > $out/bench_ref_final.json 2> $out/bench_ref_final.err
for c in 1 3 4 5 6 7 8; do
    python bench.py --config $c --steps 20 --warmup 5 > $out/bench_c$c.json 2> $out/bench_c$c.err
done
for f in $out/*.json; do
    python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d.get("roofline") or {}
print(sys.argv[1].split("/")[-1], d.get("ms_per_step"), "%.3g" % d["value"], r.get("kernel"), r.get("frac"),
      "e2e %.3g" % (d.get("e2e") or {}).get("value", 0), (d.get("cpu_baseline") or {}).get("value"),
      (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"))
PY
done
