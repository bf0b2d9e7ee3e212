"""Summarise `ncu --set full` reports (one kernel each) into a markdown table of the metrics the
roofline discussion uses: duration, DRAM bytes and throughput, tensor-pipe activity, occupancy."""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def summarise(path):
    if path.endswith(".csv"):
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    idx = {h: i for i, h in enumerate(hdr)}
    out = {"kernel": vals[idx["Kernel Name"]].split("(")[0]}
    for m, label in WANT:
        if m in idx:
            out[label] = f"{vals[idx[m]]} {units[idx[m]]}".strip()
    return out


if __name__ == "__main__":
    rs = [r for r in (summarise(p) for p in sys.argv[1:]) if r]
    cols = ["kernel"] + [l for _, l in WANT]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for r in rs:
        print("| " + " | ".join(str(r.get(c, "")) for c in cols) + " |")
