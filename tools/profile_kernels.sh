#!/bin/bash
# One plain run of tools/profile_step.py, then one `ncu --set full` capture per hot kernel
# (single launch each, inside the cudaProfilerStart/Stop range). Run under gpurun on 1 GPU.
set -u
B=${1:-16}
OUT=${2:-gpurun_out/prof_r1}
mkdir -p $OUT
python tools/profile_step.py --b $B > $OUT/plain.log 2>&1 || { echo "plain run failed"; tail $OUT/plain.log; exit 1; }
cap() {  # name regex skip
  ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:$2" -s $3 -c 1 \
      -o $OUT/$1 python tools/profile_step.py --b $B > $OUT/$1.log 2>&1
  echo "$1: $(tail -1 $OUT/$1.log)"
}
cap gemm_fc "gemm_tc_kernel" 2          # forward MLP up-projection (+bias +GELU)
cap gemm_wgrad "gemm_tc_kernel" 51      # first weight-gradient GEMM (split-K)
cap gemm_dgrad "gemm_tc_kernel" 52      # first data-gradient GEMM (+GELU backward)
cap attn_fwd "attn_fwd_kernel" 0
cap attn_bwd "attn_bwd_kernel" 0
cap adam "adam_k" 0
cap ce "ce_k" 0
cap ln_bwd "ln_bwd_rows_k" 0
ls -la $OUT
