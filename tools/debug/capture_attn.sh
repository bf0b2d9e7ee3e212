set -u
OUT=gpurun_out/r5
mkdir -p $OUT
python tools/profile_step.py --b 16 > $OUT/plain.log 2>&1 || { echo plain failed; exit 1; }
bash tools/ncu_capture.sh $OUT attn_bwd attn_bwd_kernel 3 --b 16
bash tools/ncu_capture.sh $OUT attn_fwd attn_fwd_kernel 3 --b 16
python tools/ncu_summary.py $OUT/*.raw.csv
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_v12.csv python tools/profile_step.py --b 64 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_v12.csv "v12 (b=64 micro-step, 132-SM budget)" > gpurun_out/launch_v12.md
head -16 gpurun_out/launch_v12.md
