#!/bin/bash
# C5 (Llama-style 7B, s=4096, ZeRO-3 on one rank, b=2) kernel evidence for profiles/: one plain
# run, the ncu launch list of one iteration, and `ncu --set full` captures of the LM-head GEMM (the
# step's largest forward GEMM), the gate/up GEMM, the QKV GEMM with the RoPE epilogue, both
# head_dim-128 attention kernels, the AdamW pass and the RMSNorm backward. Run under gpurun on ONE GPU.
set -u
OUT=${1:-gpurun_out/r2_c5}
ARGS="--model llama-7b --b 2 --sm 148 --stage 3"
mkdir -p $OUT
python tools/profile_step.py $ARGS > $OUT/plain.log 2>&1 || { echo "plain run failed"; tail $OUT/plain.log; exit 1; }
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/profile_step.py $ARGS > $OUT/launches.log 2>&1
python tools/launch_summary.py $OUT/launches.csv "C5 llama-7b b=2 s=4096 ZeRO-3, one rank, 148 SMs" > $OUT/launches.md
# forward order per layer: qkv, o, gate/up, down (4 GEMMs x 32 layers), then the LM head
bash tools/ncu_capture.sh $OUT gemm_lmhead "gemm_tc_kernel" 128 $ARGS
bash tools/ncu_capture.sh $OUT gemm_gateup "gemm_tc_kernel" 2 $ARGS
bash tools/ncu_capture.sh $OUT gemm_qkv_rope "gemm_tc_kernel" 0 $ARGS
bash tools/ncu_capture.sh $OUT attn_fwd "attn_fwd_d128" 0 $ARGS
bash tools/ncu_capture.sh $OUT attn_bwd "attn_bwd_d128" 0 $ARGS
bash tools/ncu_capture.sh $OUT adam "adam_k" 0 $ARGS
bash tools/ncu_capture.sh $OUT ln_bwd "ln_bwd_rows_k" 0 $ARGS
python tools/ncu_summary.py $OUT/*.raw.csv > $OUT/summary.md 2>&1
ls -la $OUT
