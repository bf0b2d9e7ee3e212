set -u
OUT=gpurun_out/r4
mkdir -p $OUT
python tools/profile_step.py --b 64 > $OUT/plain.log 2>&1 || { echo plain failed; exit 1; }
for a in "gemm_fc gemm_tc_kernel 2 64" "gemm_wgrad gemm_tc_kernel 51 64" "gemm_dgrad gemm_tc_kernel 52 64" "ce ce_smem_k 0 64" "adam adam_k 0 64" "attn_fwd attn_fwd_kernel 3 16" "attn_bwd attn_bwd_kernel 3 16" "ln_bwd ln_bwd_rows_k 0 64"; do
  set -- $a
  bash tools/ncu_capture.sh $OUT $1 $2 $3 --b $4
done
python tools/ncu_summary.py $OUT/*.raw.csv
du -sh $OUT
