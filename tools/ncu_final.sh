#!/bin/bash
# Round-2 final evidence (GPU box): ncu --set full of the current kernel of
# every BASELINE config (+ X6/X7 and C5 at the 8-way shard), each command run
# plainly first (&&) as the recipe requires; the launch list of the default
# bench; the summary JSON (tools/ncu_collect.py).  Reports other than the
# three kept ones are deleted after collection (gpurun_out size limit).
set -u
out=gpurun_out/final_ncu
mkdir -p $out
cap() { # name key kernel-regex skip [batch]
    local extra=""
    [ -n "${5:-}" ] && extra="--batch $5"
    python tools/profile_step.py $2 $extra > $out/$1.plain.log 2>&1 &&
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $out/$1 \
        python tools/profile_step.py $2 $extra > $out/$1.ncu.log 2>&1
    echo "$1 rc=$?"
}
cap c1_small_dense C1 small_dense 2
cap c2_fused C2 fused_lockstep 2
cap c3_fold_dct_f64 C3_fwd_f64 dct2_fft 2
cap c3_fold_w_i8 C3_fwd_f64 ozaki_gemmp 2
cap c3_fold_idct_f64 C3_inv_f64 idct_fft 2
cap c3_fold_wt_i8 C3_inv_f64 ozaki_gemmp 2
cap c3f_fold_dct C3_fwd_f32 dct2_fft 2
cap c3f_split C3_fwd_f32 bf16x3_split 2
cap c3f_fold_w_bf16x3 C3_fwd_f32 tc_bf16x3_kernel 2
cap c3f_fold_idct C3_inv_f32 idct_fft 2
cap c3f_fold_wt_bf16x3 C3_inv_f32 tc_bf16x3_kernel 2
cap c4_split C4 bf16x3_split 2
cap c4_bf16x3 C4 tc_bf16x3_kernel 2
cap c5_slice C5 ozaki_slice 2
cap c5_dense_i8 C5 ozaki_gemm2 2
cap c5_dense_i8_256rows C5 ozaki_gemm2 2 256
cap x6_chain_i8 X6 ozaki_gemm 2
cap x7_nfst_i8 X7 ozaki_gemm 2
cap x8_slice X8 ozaki_slice 2
python tools/ncu_collect.py $out $out/ncu_summary_final.json > $out/collect.log 2>&1; echo "collect rc=$?"
for f in $out/*.ncu-rep; do
    case $(basename $f) in c5_dense_i8.ncu-rep|c3_fold_w_i8.ncu-rep|c4_bf16x3.ncu-rep) ;; *) rm -f $f ;; esac
done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs --sustain-s 0 > $out/bench_plain.json 2> $out/bench_plain.err &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bench_c5.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs --sustain-s 0 > $out/bench_ncu.log 2>&1
echo "launches rc=$?"
