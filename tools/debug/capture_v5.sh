# ncu --set full captures (one launch each) of the round-1 final kernels -> gpurun_out/r5ncu
set -u
OUT=gpurun_out/r5ncu
mkdir -p $OUT
python tools/profile_step.py --b 64 > $OUT/plain.log 2>&1 || { echo plain failed; exit 1; }
for a in "gemm_fc gemm_tc_kernel 2 64" "gemm_dgrad_gelu gemm_tc_kernel 52 64" "gemm_wgrad gemm_tc_kernel 51 64" "ce ce_reg_k 0 64" "ln_bwd ln_bwd_fused_k 1 64" "attn_fwd attn_fwd_kernel 3 16" "attn_bwd attn_bwd_kernel 3 16"; do
  set -- $a
  timeout 900 bash tools/ncu_capture.sh $OUT $1 $2 $3 --b $4
done
python tools/ncu_summary.py $OUT/*.raw.csv > $OUT/summary.md 2>&1
cat $OUT/summary.md
du -sh $OUT
