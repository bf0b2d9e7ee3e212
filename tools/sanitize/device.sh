#!/bin/bash
# compute-sanitizer passes (memcheck, racecheck, synccheck) over small cases of the kernel parity
# tests: the tcgen05 GEMM (both operand majors, fused epilogues), fused attention fwd/bwd at
# head_dim 64 and 128, the single-device peer collectives (mbarrier / flag protocols), and one
# tiny ZeRO-3 step. Run under gpurun on ONE GPU. Logs: OUT/<tool>.log (summary line at the end).
set -u
OUT=${1:-gpurun_out/r2_sanitizer}
mkdir -p "$OUT"
CS=${CS:-compute-sanitizer}
SEL_GEMM="tests/test_gemm_gpu.py::test_gemm_majors tests/test_gemm_gpu.py::test_gemm_bias_resid_gelu"
SEL_ATTN="tests/test_attention_gpu.py -k fwd_bwd and 1-128-1-0 or 1-256-2-0"
run() {  # tool, name, pytest args...
  local tool=$1 name=$2; shift 2
  timeout 1500 $CS --tool "$tool" --target-processes all --print-limit 20 \
      python -m pytest -x -q -p no:cacheprovider "$@" > "$OUT/$tool.$name.log" 2>&1
  echo "$tool $name rc=$? :: $(grep -E 'ERROR SUMMARY|passed|failed' "$OUT/$tool.$name.log" | tail -2 | tr '\n' ' ')"
}
for tool in memcheck racecheck synccheck; do
  run $tool gemm tests/test_gemm_gpu.py -k "majors and (128-64-64 or 256-256-128) or bias_resid_gelu and 256-768-256"
  run $tool attn tests/test_attention_gpu.py -k "(fwd_bwd and (1-128-1-0 or 1-256-2-0)) and not perf"
  run $tool peer tests/test_peer_gpu.py -k "[2] or 2-False"
  run $tool step tests/test_step_gpu.py -k "test_step_matches_fp64_oracle and 3-4-4-1"
done
