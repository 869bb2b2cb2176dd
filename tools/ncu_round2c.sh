#!/bin/bash
# Round-2 (third batch) ncu captures: the int8 products after the split-K
# tail and the batched TMEM epilogue (C3 fp64 forward / inverse, the rank-k
# chain X6, C5 at full batch and at the 8-way shard's 256 rows).
set -u
out=gpurun_out/ncu4
mkdir -p $out
cap() { # name key kernel-regex skip [batch]
    local extra=""
    [ -n "${5:-}" ] && extra="--batch $5"
    python tools/profile_step.py $2 $extra > $out/$1.plain.log 2>&1 &&
    ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $out/$1 \
        python tools/profile_step.py $2 $extra > $out/$1.ncu.log 2>&1
    echo "$1 rc=$?"
}
cap c3_fold_w_i8 C3_fwd_f64 ozaki_gemm 2
cap c3_fold_wt_i8 C3_inv_f64 ozaki_gemm 2
cap c5_dense_i8 C5 ozaki_gemm 2
cap c5_dense_i8_256 C5 ozaki_gemm 2 256
