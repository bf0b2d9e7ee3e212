# A/B two builds on one box: build A, copy it to alt_lib/libA.so, rebuild B (working tree), then
#   gpurun -- bash tools/debug/ab.sh
# A/B of two builds on the same box: B = working tree (tests first), A = alt_lib/libA.so
set -u
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_step_gpu.py -x -q > gpurun_out/ab/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab/pytest.log
python tools/profile_step.py --b 64 > gpurun_out/ab/plain.log 2>&1 || { echo plain failed; tail gpurun_out/ab/plain.log; exit 1; }
cp paper_2408_12596_b200/lib/libzp.so alt_lib/libB.so
for v in B A B2 A2; do
  case $v in A|A2) cp alt_lib/libA.so paper_2408_12596_b200/lib/libzp.so;; *) cp alt_lib/libB.so paper_2408_12596_b200/lib/libzp.so;; esac
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab/l_$v.csv python tools/profile_step.py --b 64 > gpurun_out/ab/ncu_$v.log 2>&1
  python tools/launch_summary.py gpurun_out/ab/l_$v.csv "$v" > gpurun_out/ab/l_$v.md
  echo "== $v"; grep -E "launches,|ce_|gemm_tc_kernel<256, 0, 0" gpurun_out/ab/l_$v.md
done
cp alt_lib/libB.so paper_2408_12596_b200/lib/libzp.so
