# fused LayerNorm backward variants (shared-memory atomics vs register accumulators): launch lists
set -u
mkdir -p gpurun_out/r7
timeout 600 python -m pytest tests/test_step_gpu.py -x -q 2>&1 | tail -2
ZP_LNB_REG=1 timeout 600 python -m pytest tests/test_step_gpu.py -x -q 2>&1 | tail -2
python tools/profile_step.py --b 64 > gpurun_out/r7/plain.log 2>&1 || { echo plain failed; tail gpurun_out/r7/plain.log; exit 1; }
for m in smem reg; do
  if [ $m = reg ]; then export ZP_LNB_REG=1; fi
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ln_bwd --csv --log-file gpurun_out/r7/ln_$m.csv python tools/profile_step.py --b 64 > gpurun_out/r7/ncu_$m.log 2>&1
  python - gpurun_out/r7/ln_$m.csv $m <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); agg[d["Kernel Name"].split("(")[0]][d["Metric Name"] + " " + d["Metric Unit"]].append(float(d["Metric Value"].replace(",", "")))
for k, m in agg.items():
    print(sys.argv[2], k[:60], {n: (len(v), round(sum(v) / len(v), 2)) for n, v in m.items()})
PY
done
