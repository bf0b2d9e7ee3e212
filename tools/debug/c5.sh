# C5 (Llama-style 7B, s4096, ZeRO-3) on 4 emulated heterogeneous ranks.
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 bench.py --config c5 --gpus 4 --steps 2 --warmup 3 > gpurun_out/bench_c5_n4.json 2> gpurun_out/bench_c5_n4.err
echo rc=$?
tail -5 gpurun_out/bench_c5_n4.err
python -c "
import json
l=[x for x in open('gpurun_out/bench_c5_n4.json') if x.startswith('{')]
d=json.loads(l[-1])
print(round(d['value'],2), d['config']['plan'], d['config'].get('mbs'), 'uniform', round(d['uniform_split']['value'],2), round(d['uniform_split']['poplar_speedup'],3), 'idle', [round(x,2) for x in d['sync_idle_pct']], 'gemm', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), d['ms_per_step'])
"
