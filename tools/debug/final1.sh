# Round-end style check on one GPU: full GPU test suite, smoke, default bench, launch list.
set -u
mkdir -p gpurun_out/f1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f1/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/f1/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/f1/smoke.log
timeout 900 python bench.py > gpurun_out/f1/bench.json 2> gpurun_out/f1/bench.err; echo "bench rc=$?"
python -c "
import json
l=[x for x in open('gpurun_out/f1/bench.json') if x.startswith('{')]
d=json.loads(l[-1])
print(round(d['value'],1), d['config']['plan'], 'gemm', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'], d['cpu_baseline']['value'] if d.get('cpu_baseline') else None, d['gpu_launches'])
"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f1/bench_ref.json 2> gpurun_out/f1/bench_ref.err; echo "ref rc=$?"; tail -c 400 gpurun_out/f1/bench_ref.json
python tools/profile_step.py --b 64 > gpurun_out/f1/plain.log 2>&1 || { echo plain failed; exit 1; }
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f1/launch.csv python tools/profile_step.py --b 64 > gpurun_out/f1/ncu.log 2>&1
python tools/launch_summary.py gpurun_out/f1/launch.csv "v16 (b=64 micro-step, 132-SM budget)" > gpurun_out/f1/launch.md
head -24 gpurun_out/f1/launch.md
