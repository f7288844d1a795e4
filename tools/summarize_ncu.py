"""Summarise ncu outputs for profiles/: launch list (per-kernel share of device time) and a
--set full report (per-launch DRAM bytes, throughput, occupancy, registers).

    python tools/summarize_ncu.py launches <launches.csv>
    python tools/summarize_ncu.py full <report.ncu-rep>
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, ni, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in data:
        if len(r) <= vi or r[ni] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        agg[r[ki].split("(")[0]][0] += 1
        agg[r[ki].split("(")[0]][1] += v
        tot += v
    print(f"# ncu launch list ({path}): gpu__time_duration.sum, cold-cache serialised; total {tot / 1e6:.3f} ms")
    print(f"{'ms':>10} {'share':>6} {'launches':>8} {'us/launch':>10}  kernel")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v / 1e6:10.3f} {100 * v / tot:5.1f}% {c:8d} {v / c / 1e3:10.1f}  {k}")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    idx = [(w, hdr.index(w)) for w in WANT if w in hdr]
    print(f"# ncu --set full ({path})")
    print("kernel | " + " | ".join(f"{w} [{units[i]}]" for w, i in idx))
    for r in rows[2:]:
        print(r[ki].split("(")[0] + " | " + " | ".join(r[i] for _, i in idx))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
