"""Per-block timeline of one attention-backward launch (build with
NVFLAGS_EXTRA=-DDH_ATTN_BLKTRACE): makespan, per-SM busy time, the critical
SM's items. usage: attn_blocks.py <nq> [T] [fwd]; env DH_ATTN_FWD_CHUNK forces the forward KV chunk"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh
nq = int(sys.argv[1]) if len(sys.argv) > 1 else 4
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
fwd_only = len(sys.argv) > 3 and sys.argv[3] == "fwd"
nkv, d = max(1, nq // 4), 128
qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda") * 0.5).to(torch.bfloat16)
q, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nq, T, device="cuda")
do = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
for _ in range(3):
    dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, d ** -0.5)
    if fwd_only:
        continue
    dh.attn_bwd(q, k, v, o, lse, do, dqkv[:, :nq * d], dqkv[:, nq * d:(nq + nkv) * d], dqkv[:, (nq + nkv) * d:],
                nq, nkv, d, d ** -0.5)
torch.cuda.synchronize()
n = 8192
buf = (ctypes.c_ulonglong * (n * 3))()
dh.lib().dh_attn_blk_read(buf, n * 3)
rows = [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n) if buf[3 * i] and buf[3 * i + 1] >= buf[3 * i]]
t0 = min(r[0] for r in rows)
t1 = max(r[1] for r in rows)
print(f"{len(rows)} blocks, makespan {(t1 - t0) / 1e3:.1f} us")
busy = {}
for s0, e0, sm in rows:
    busy.setdefault(sm, []).append(((s0 - t0) / 1e3, (e0 - t0) / 1e3))
tot = sum(e - s for v in busy.values() for s, e in v)
print(f"SMs used {len(busy)}, mean busy {tot / len(busy):.1f} us, idle fraction {1 - tot / (len(busy) * (t1 - t0) / 1e3):.3f}")
dur = sorted(((e0 - s0) / 1e3, i) for i, (s0, e0, sm) in enumerate(rows))
print("longest items (us):", [round(x[0], 1) for x in dur[-8:]])
print("first-start / last-start (us):", round(min(r[0] - t0 for r in rows) / 1e3, 2),
      round(max(r[0] - t0 for r in rows) / 1e3, 2))
ends = sorted((max(e for s, e in v), sm) for sm, v in busy.items())
print("SM finish times (us): min %.1f median %.1f max %.1f" % (ends[0][0], ends[len(ends) // 2][0], ends[-1][0]))
crit = ends[-1][1]
print("critical SM items:", [(round(s, 1), round(e, 1)) for s, e in sorted(busy[crit])])
cnt = {}
for sm, v in busy.items():
    cnt.setdefault(len(v), []).append(sum(e - s for s, e in v))
print("items per SM -> (SMs, mean busy us, max busy us):",
      {k: (len(v), round(sum(v) / len(v), 1), round(max(v), 1)) for k, v in sorted(cnt.items())})
print("item durations (us) deciles:", [round(dur[int(i * (len(dur) - 1) / 10)][0], 1) for i in range(11)])
if fwd_only and hasattr(dh.lib(), "dh_attn_phase_read"):
    ph = (ctypes.c_ulonglong * (n * 8))()
    dh.lib().dh_attn_phase_read(ph, n * 8)
    names = ["prologue done", "Q + K_0 landed", "first S_0 ready", "tile 0 O done", "partials issued", "block end"]
    rel = {k: [] for k in names}
    for i in range(n):
        s0, e0 = buf[3 * i], buf[3 * i + 1]
        if not s0 or e0 < s0:
            continue
        vals = [ph[8 * i + j] for j in range(5)] + [e0]
        for k, v in zip(names, vals):
            if v >= s0:
                rel[k].append((v - s0) / 1e3)
    print("forward phases, us after block start (median / p90):")
    for k, v in rel.items():
        if v:
            v.sort()
            print(f"  {k:18s} {v[len(v) // 2]:6.2f} / {v[int(0.9 * (len(v) - 1))]:6.2f}  ({len(v)} blocks)")
