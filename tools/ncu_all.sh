#!/bin/bash
# ncu --set full captures of every kernel the BASELINE configs run (one launch
# each, after warm-up launches), plus the launch list of the default bench.
# Each profiled command first runs once plainly (&&) as the recipe requires.
set -u
out=gpurun_out/ncu
mkdir -p $out
cap() { # name key kernel-regex skip
    python tools/profile_step.py $2 > $out/$1.plain.log 2>&1 &&
    ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $out/$1 \
        python tools/profile_step.py $2 > $out/$1.ncu.log 2>&1
    echo "$1 rc=$?"
}
cap c1_fused C1 fused 2
cap c2_fused C2 fused 2
cap c3_fold_dct_f64 C3_fwd_f64 dct2_fft 3
cap c3_fold_w_f64 C3_fwd_f64 rows_by_basis 2
cap c3_fold_idct_f64 C3_inv_f64 idct_fft 3
cap c3_fold_wt_f64 C3_inv_f64 rows_by_basis 3
cap c3_fold_w_tc32 C3_fwd_f32 tc_sgemm3 2
cap c3_fold_wt_tc32 C3_inv_f32 tc_sgemm3 3
cap c4_tc32 C4 tc_sgemm3 2
cap c5_slice C5 ozaki_slice 3
cap c5_dense_i8 C5 ozaki_gemm 2
cap x6_chain_i8 X6 ozaki_gemm 2
cap x7_nfst_fwd X7 nfst_forward 2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs --sustain-s 0 > $out/bench_plain.json 2> $out/bench_plain.err &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bench_c5.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs --sustain-s 0 > $out/bench_ncu.log 2>&1
echo "launches rc=$?"
