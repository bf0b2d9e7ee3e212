set -u
mkdir -p gpurun_out/r9
timeout 600 python -m pytest tests/test_step_gpu.py -x -q 2>&1 | tail -2
python tools/profile_step.py --b 64 > gpurun_out/r9/plain.log 2>&1 || { echo plain failed; tail gpurun_out/r9/plain.log; exit 1; }
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:ln_bwd --csv --log-file gpurun_out/r9/ln.csv python tools/profile_step.py --b 64 > gpurun_out/r9/ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r9/ln.csv "ln" | tail -3
python tools/profile_step.py --b 64 --model gpt2-medium --stage 2 > gpurun_out/r9/plain_m.log 2>&1 || { echo plain medium failed; tail gpurun_out/r9/plain_m.log; }
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:ln_bwd --csv --log-file gpurun_out/r9/ln_m.csv python tools/profile_step.py --b 32 --model gpt2-medium > gpurun_out/r9/ncu_m.log 2>&1
python tools/launch_summary.py gpurun_out/r9/ln_m.csv "ln medium b32" | tail -3
