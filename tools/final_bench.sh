#!/bin/bash
# End-of-round bench set (GPU box) into gpurun_out/final/: the default bench
# line (C5 headline + every BASELINE config), the reference arm, the SURVEY
# 8(f) extras (X6 chain, X7 / X8 NFST route), the C5 shard sweep, clocks.
set -u
out=gpurun_out/final
mkdir -p $out
python bench.py > $out/bench_final.json 2> $out/bench_final.err; echo "bench rc=$?"
python bench.py --impl reference > $out/bench_ref_final.json 2> $out/bench_ref_final.err; echo "reference rc=$?"
for c in X6 X7 X8; do
    python bench.py --config $c --no-configs --steps 20 --warmup 5 > $out/bench_$c.json 2> $out/bench_$c.err
    echo "$c rc=$?"
done
python tools/shard_sweep.py > $out/shard_sweep.jsonl 2>&1; echo "shard sweep rc=$?"
