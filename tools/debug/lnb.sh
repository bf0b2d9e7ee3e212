# fused LayerNorm backward: step parity, then a launch list of one b=64 GPT-2 micro-step and the N=1 bench
set -u
timeout 900 python -m pytest tests/test_step_gpu.py -x -q 2>&1 | tail -3
mkdir -p gpurun_out/r6
python tools/profile_step.py --b 64 > gpurun_out/r6/plain.log 2>&1 || { echo plain failed; tail gpurun_out/r6/plain.log; exit 1; }
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6/launch.csv python tools/profile_step.py --b 64 > gpurun_out/r6/ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r6/launch.csv "v13 (b=64 micro-step, 132-SM budget)" > gpurun_out/r6/launch.md
head -25 gpurun_out/r6/launch.md
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6/bench.json 2> gpurun_out/r6/bench.err
python -c "
import json
l=[x for x in open('gpurun_out/r6/bench.json') if x.startswith('{')]
d=json.loads(l[-1])
print(round(d['value'],1), d['config']['plan'], 'gemm', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'])
"
