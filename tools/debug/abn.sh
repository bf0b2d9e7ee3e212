# A/B/.. of prebuilt libraries alt_lib/lib_*.so on one box (attention parity for each, then the launch list)
set -u
mkdir -p gpurun_out/abn
python tools/profile_step.py --b 64 > gpurun_out/abn/plain.log 2>&1 || { echo plain failed; tail gpurun_out/abn/plain.log; exit 1; }
for rep in 1 2; do
for f in alt_lib/lib_*.so; do
  v=$(basename $f .so)_$rep
  cp $f paper_2408_12596_b200/lib/libzp.so
  if [ $rep = 1 ]; then timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_step_gpu.py -x -q > gpurun_out/abn/pt_$v.log 2>&1; echo "$v pytest rc=$? $(tail -1 gpurun_out/abn/pt_$v.log)"; fi
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/abn/l_$v.csv python tools/profile_step.py --b 64 > gpurun_out/abn/ncu_$v.log 2>&1
  python tools/launch_summary.py gpurun_out/abn/l_$v.csv "$v" > gpurun_out/abn/l_$v.md
  echo "== $v $(grep -E 'launches,' gpurun_out/abn/l_$v.md)"; grep -E "${ABN_GREP:-attn_fwd}" gpurun_out/abn/l_$v.md
done
done
