# ZeRO-3 gather prefetch check: multi-GPU parity, then the Z3 benches on 4 GPUs.
timeout 900 python -m pytest tests/test_multigpu_gpu.py -x -q 2>&1 | tail -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29630 bench.py --config c3 --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_c3_n4.json 2> gpurun_out/bench_c3_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640 bench.py --config c4 --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_c4_n4.json 2> gpurun_out/bench_c4_n4.err
for f in bench_c3_n4 bench_c4_n4; do
python -c "
import json
l=[x for x in open('gpurun_out/$f.json') if x.startswith('{')]
if not l: print('$f', 'NO LINE'); raise SystemExit
d=json.loads(l[-1])
print('$f', round(d['value'],1), d['config']['plan'], 'uniform', round(d['uniform_split']['value'],1), round(d['uniform_split']['poplar_speedup'],3), 'idle', [round(x,2) for x in d['sync_idle_pct']], 'e2e', round(d['e2e']['value'],1))
"
tail -3 gpurun_out/$f.err
done
