set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_n1_full.json 2> gpurun_out/bench_n1_full.err; tail -c 3000 gpurun_out/bench_n1_full.json
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  tail -c 600 gpurun_out/bench_n$N.json
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29520 bench.py --config c3 --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_c3_n4.json 2> gpurun_out/bench_c3_n4.err
tail -c 600 gpurun_out/bench_c3_n4.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -c 800 gpurun_out/bench_ref.json
