# fused LayerNorm backward (two rows per warp): parity, ln_bwd timing for min-blocks 2 vs 3
set -u
mkdir -p gpurun_out/r8
timeout 600 python -m pytest tests/test_step_gpu.py -x -q 2>&1 | tail -2
python tools/profile_step.py --b 64 > gpurun_out/r8/plain.log 2>&1 || { echo plain failed; tail gpurun_out/r8/plain.log; exit 1; }
for m in minb2 minb3; do
  if [ $m = minb3 ]; then cp alt_lib/libzp_minb3.so paper_2408_12596_b200/lib/libzp.so; fi
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:ln_bwd --csv --log-file gpurun_out/r8/ln_$m.csv python tools/profile_step.py --b 64 > gpurun_out/r8/ncu_$m.log 2>&1
  python tools/launch_summary.py gpurun_out/r8/ln_$m.csv "$m" | tail -3
done
