# Multi-GPU: peer-collective parity tests (2 and 4 ranks), C2 at N=2 and N=4, reference arm at N=4.
set -u
timeout 900 python -m pytest tests/test_multigpu_gpu.py -x -q 2>&1 | tail -2
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  echo "N=$N rc=$?"
  python -c "
import json
l=[x for x in open('gpurun_out/bench_n$N.json') if x.startswith('{')]
d=json.loads(l[-1])
print('N=$N', round(d['value'],1), d['config']['plan'], 'uniform', round(d['uniform_split']['value'],1), round(d['uniform_split']['poplar_speedup'],3), 'idle', [round(x,2) for x in d['sync_idle_pct']], 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])
"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29790 bench.py --impl reference --gpus 4 --steps 2 --warmup 3 > gpurun_out/bench_ref_n4.json 2> gpurun_out/bench_ref_n4.err
echo "ref N=4 rc=$?"; grep -c '^{' gpurun_out/bench_ref_n4.json
