#!/bin/bash
# Second batch of round-2 ncu captures: the kernels added or rerouted after
# tools/ncu_all.sh ran (small dense C1, int8 fold product C3 fp64, bf16x3 fold
# products C3 fp32, the slicing / split passes, the per-graph setup kernels).
set -u
out=gpurun_out/ncu3
mkdir -p $out
cap() { # name key kernel-regex skip
    python tools/profile_step.py $2 > $out/$1.plain.log 2>&1 &&
    ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $out/$1 \
        python tools/profile_step.py $2 > $out/$1.ncu.log 2>&1
    echo "$1 rc=$?"
}
cap c1_small_dense C1 small_dense 2
cap c3_fold_w_i8 C3_fwd_f64 ozaki_gemm 2
cap c3_slice_fold C3_fwd_f64 ozaki_slice 3
cap c3f_fold_w_bf16x3 C3_fwd_f32 tc_bf16x3_kernel 2
cap c3f_fold_wt_bf16x3 C3_inv_f32 tc_bf16x3_kernel 2
cap c3f_fold_dct C3_fwd_f32 dct2_fft 2
cap c4_split C4 bf16x3_split 2
cap c5_secular C5 secular_roots 0
cap c5_normalisers C5 normalisers 0
cap c5_column_signs C5 column_signs 0
