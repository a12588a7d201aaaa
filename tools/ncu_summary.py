"""Summarise an ncu report: key metrics + top stall PCs (SASS) -> stdout."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__cluster_dim_x",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    print("kernel:", r[h.index("Kernel Name")][:80])
    for k in keys:
        for i, name in enumerate(h):
            if name == k or name.endswith("." + k):
                print(f"  {k} = {r[i]} {u[i]}")
                break
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    hh = srows[1]
    i_s = hh.index("Warp Stall Sampling (All Samples)")
    i_src = hh.index("Source")
    i_ex = hh.index("Instructions Executed")
    data = []
    for r in srows[2:]:
        try:
            data.append((int(r[i_s] or 0), r[0][-5:], r[i_src][:90], r[i_ex]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    print("top stall PCs (samples, %, pc, sass, executed):")
    for d in sorted(data, reverse=True)[: int(sys.argv[2])]:
        print(f"  {d[0]:8d} {100*d[0]/tot:5.1f}% {d[1]} {d[2]} | {d[3]}")
