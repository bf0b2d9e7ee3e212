set -u
timeout 900 python -m pytest tests/test_multigpu_gpu.py -x -q 2>&1 | tail -2
mkdir -p gpurun_out/nvl
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2981$N tools/nvlink_bench.py --out gpurun_out/nvl/nvlink_n$N.json > gpurun_out/nvl/n$N.log 2>&1
  echo "N=$N rc=$?"; cat gpurun_out/nvl/nvlink_n$N.json 2>/dev/null || tail -20 gpurun_out/nvl/n$N.log
done
