set -u
mkdir -p gpurun_out/r10
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py -x -q 2>&1 | tail -2
python tools/profile_step.py --b 64 > gpurun_out/r10/plain.log 2>&1 || { echo plain failed; tail gpurun_out/r10/plain.log; exit 1; }
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r10/launch.csv python tools/profile_step.py --b 64 > gpurun_out/r10/ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r10/launch.csv "v14 (b=64 micro-step, 132-SM budget)" > gpurun_out/r10/launch.md
head -26 gpurun_out/r10/launch.md
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r10/bench.json 2> gpurun_out/r10/bench.err
python -c "
import json
l=[x for x in open('gpurun_out/r10/bench.json') if x.startswith('{')]
d=json.loads(l[-1])
print(round(d['value'],1), d['config']['plan'], 'gemm', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'])
"
