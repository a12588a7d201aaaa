"""Summarise an ncu report: key metrics + top stall PCs (SASS) -> stdout.

  python tools/ncu_summary.py REPORT [N_PCS] [--lines N] [--stalls]
    N_PCS     top-N SASS instructions by warp-stall samples
    --lines N top-N CUDA source lines (file:line) by stall samples; an inlined instruction
              counts under every line of its inline chain, so shares overlap
    --stalls  stall-reason breakdown (share of all samples)
"""
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
args = sys.argv[2:]
lines_n = int(args[args.index("--lines") + 1]) if "--lines" in args else 0
want_stalls = "--stalls" in args
pcs = [a for i, a in enumerate(args) if a.isdigit() and (i == 0 or args[i - 1] != "--lines")]
if lines_n or want_stalls:
    import collections
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "sass,cuda"], capture_output=True, text=True).stdout
    by, text, stalls = collections.Counter(), {}, collections.Counter()
    f = h = None
    key = None
    for r in csv.reader(io.StringIO(src)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            h = r
            i_s = h.index("Warp Stall Sampling (All Samples)")
            st_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
            continue
        if h is None or len(r) <= i_s:
            continue
        if r[0]:
            key = (f, int(r[0]))
            text[key] = r[1][:90]
        try:
            by[key] += int(r[i_s] or 0)
            for i in st_cols:
                stalls[h[i][6:]] += int(r[i] or 0)
        except ValueError:
            pass
    tot = sum(by.values()) or 1
    if want_stalls:
        # from the SASS-only page: the sass+cuda page repeats an inlined instruction's samples
        # under every source file of its inline chain
        sp = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                             "sass"], capture_output=True, text=True).stdout
        srows = list(csv.reader(io.StringIO(sp)))
        hs = srows[1] if srows[1] and srows[1][0] == "Address" else srows[0]
        cols = [i for i, n in enumerate(hs) if n.startswith("stall_") and "Not Issued" not in n]
        stalls = collections.Counter()
        for r in srows[2:]:
            if len(r) < len(hs):
                continue
            for i in cols:
                try:
                    stalls[hs[i][6:]] += int(r[i] or 0)
                except ValueError:
                    pass
        st_tot = sum(stalls.values()) or 1
        print("stall reasons:", ", ".join(f"{k} {100 * v / st_tot:.1f}%" for k, v in stalls.most_common(8)))
    if lines_n:
        print("top source lines (samples, %, file:line, source):")
        for k, v in by.most_common(lines_n):
            print(f"  {v:8d} {100 * v / tot:5.1f}% {k[0]}:{k[1]} {text.get(k, '')}")
if pcs:
    sys.argv = sys.argv[:2] + [pcs[0]]
if len(sys.argv) > 2 and sys.argv[2].isdigit():
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
