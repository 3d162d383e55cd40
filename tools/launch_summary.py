"""Summarise an ncu --metrics gpu__time_duration.sum CSV: time share per kernel."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi: continue
    name = r[ki]
    short = re.sub(r"\(.*", "", name)
    short = re.sub(r"^void ", "", short)
    m = re.search(r"gemm_tcgen05_kernel<(\d+), (\w+), (\w+), (\w+)>", name)
    if m: short = f"gemm<BN{m.group(1)},A_MN={m.group(2)},B_MN={m.group(3)},F32={m.group(4)}>"
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    us = v / 1000 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1000
    agg[short][0] += 1; agg[short][1] += us
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{100*us/tot:6.2f}%  {us:10.1f} us  {n:5d}x  {k[:110]}")
