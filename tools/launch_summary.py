"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into a markdown table
(kernel, launches, total time, share of the profiled range)."""
import collections
import csv
import sys


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"]
        name = name.split("(")[0] if "gemm_tc_kernel" not in name else name.split("(")[0]
        name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"### {title}\n\n{len(data)} launches, {tot / 1e3:.2f} ms total (serialised, cold-cache ncu times)\n")
    print("| kernel | launches | total ms | share |\n|---|---:|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {v[0]} | {v[1] / 1e3:.3f} | {100 * v[1] / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
