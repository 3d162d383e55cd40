"""Summarise an ncu capture of tools/hbm_kernels.py against MEASURED_PEAKS.json:

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/hbm.csv python tools/hbm_kernels.py > gpurun_out/hbm.json
  python tools/hbm_summary.py gpurun_out/hbm.csv gpurun_out/hbm.json

Achieved GB/s = algorithmic bytes per launch / kernel duration; frac against
the measured HBM copy bandwidth (burst: each kernel is timed alone)."""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(io.StringIO(open(sys.argv[1]).read())))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
expect = json.loads([x for x in open(sys.argv[2]) if x.startswith("{")][-1])["algorithmic_bytes_per_launch"]
pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
kern = {}
for r in rows[start + 1:]:
    if len(r) != len(h):
        continue
    name, metric, val = r[h.index("Kernel Name")], r[h.index("Metric Name")], r[h.index("Metric Value")]
    unit = r[h.index("Metric Unit")]
    key = (r[h.index("ID")], name)
    v = float(val.replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "byte": 1e-6, "B": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3,
             "GB": 1e3}.get(unit, 1.0)
    kern.setdefault(key, {})[metric] = v * scale
match = {"rmsnorm_fwd": "rmsnorm_fwd", "rmsnorm_bwd": "rmsnorm_bwd", "add_kernel": "add", "swiglu_fwd": "swiglu_fwd",
         "swiglu_bwd": "swiglu_bwd", "rope": "rope", "adamw": "adamw"}
print(f"HBM-bound kernels, TP=1 Llama-3-8B shapes, one launch each, ncu --clock-control none; "
      f"peak {pk} GB/s (MEASURED_PEAKS.json hbm_gbs)")
print(f"{'kernel':45s} {'us':>8s} {'algo MB':>9s} {'algo GB/s':>10s} {'frac':>6s} {'dram MB':>9s}")
for (kid, name), m in kern.items():
    if "dh::" not in name:  # torch's input initialisation
        continue
    base = next((v for k, v in match.items() if k in name), None)
    us = m.get("gpu__time_duration.sum", 0.0)
    dram = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    if base is None:
        print(f"{name[:45]:45s} {us:8.1f} {'-':>9s} {'-':>10s} {'-':>6s} {dram:9.1f}")
        continue
    mb = expect[base] / 1e6
    gbs = mb / us * 1e3
    print(f"{name[:45]:45s} {us:8.1f} {mb:9.1f} {gbs:10.0f} {gbs / pk:6.2f} {dram:9.1f}")
