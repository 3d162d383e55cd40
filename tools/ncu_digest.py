"""Digest of an ncu --set full report: duration, clocks, pipe utilisation,
top stall reasons and the hottest SASS instructions (ncu -i ... --csv)."""
import csv, subprocess, sys, io

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
args = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["--kernel-name", f"regex:{kern}"] if kern else [])
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
h, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"]
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")][:80])
    for k in keys:
        if k in h:
            print(f"  {k:80s} {r[h.index(k)]} {units[h.index(k)]}")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(r[i]), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("  stalls per issue:", ", ".join(f"{k} {v:.2f}" for v, k in sorted(st, reverse=True)[:8]))
if len(sys.argv) > 3:
    args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + (["--kernel-name", f"regex:{kern}"] if kern else [])
    rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
    hh = rows[1]
    si = hh.index("Warp Stall Sampling (All Samples)")
    data = []
    seen = set()
    for r in rows[2:]:
        try:
            if r[0] in seen:
                continue
            seen.add(r[0])
            data.append((int(r[si]), r[1]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    for v, src in sorted(data, reverse=True)[:int(sys.argv[3])]:
        print(f"  {100 * v / tot:5.1f}%  {src[:100]}")
