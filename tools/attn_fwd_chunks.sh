for c in 0 4 6 8 10 12 16; do
  if [ $c = 0 ]; then unset DH_ATTN_FWD_CHUNK; else export DH_ATTN_FWD_CHUNK=$c; fi
  python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2411_15871_b200 import device as dh
T, nq, nkv, d = 4096, 4, 1, 128
qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda") * 0.5).to(torch.bfloat16)
q, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16); lse = torch.empty(nq, T, device="cuda")
n = dh.attn_fwd_scratch_floats(T, nq, nkv, d)
sc = torch.empty(max(n, 1), device="cuda")
def f():
    dh.lib().dh_attn_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), q.stride(0), k.stride(0), o.data_ptr(), o.stride(0), lse.data_ptr(), sc.data_ptr() if n else None, n, T, nq, nkv, d, d ** -0.5, torch.cuda.current_stream().cuda_stream)
for _ in range(3): f()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(50): f()
e.record(); torch.cuda.synchronize()
print(os.environ.get("DH_ATTN_FWD_CHUNK", "auto"), n, round(s.elapsed_time(e) / 50 * 1e3, 1), "us")
PY
done
