"""Launch one kernel of interest a few times (for ncu --set full captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh
which = sys.argv[1] if len(sys.argv) > 1 else "gemm_tp1"
if which.startswith("gemm"):
    shapes = {"gemm_tp1": (4096, 14336, 4096), "gemm_tp8": (4096, 1792, 4096),
              "gemm_proj8": (4096, 4096, 512), "gemm_qkv8": (4096, 768, 4096)}
    m, n, k = shapes[which]
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        dh.gemm(a, b, d)
elif which.startswith("wgrad"):
    # mlp_fc1_wgrad's GEMM: dW[F,H] += d_gate^T ln1 (A and B MN-major, fp32 reduce-add)
    S, H, F = 4096, 4096, 14336 if which.endswith("tp1") else 1792
    a = torch.randn(S, F, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(S, H, device="cuda", dtype=torch.bfloat16)
    d = torch.zeros(F, H, device="cuda", dtype=torch.float32)
    for _ in range(3):
        dh.gemm(a, b, d, a_mn=True, b_mn=True, accumulate=True)
elif which.startswith("swiglu"):
    m, n, k = (4096, 14336, 4096) if which.endswith("tp1") else (4096, 1792, 4096)
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    d, d2, aux0, aux1 = (torch.randn(m, n, device="cuda").to(torch.bfloat16) for _ in range(4))
    epi = dh.EPI_SWIGLU_BWD if "bwd" in which else dh.EPI_SWIGLU_FWD
    for _ in range(3):
        dh.gemm(a, b, d, epilogue=epi, d2=d2, aux0=aux0, aux1=aux1)
elif which.startswith("attn"):
    T, nq, nkv, D = (4096, 32, 8, 128) if which == "attn_tp1" else (4096, 4, 1, 128)
    qkv = (torch.randn(T, (nq + 2 * nkv) * D, device="cuda") * 0.5).to(torch.bfloat16)
    q, k_, v = qkv[:, :nq * D], qkv[:, nq * D:(nq + nkv) * D], qkv[:, (nq + nkv) * D:]
    o = torch.empty(T, nq * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    for _ in range(3):
        dh.attn_fwd(q, k_, v, o, lse, nq, nkv, D, D ** -0.5)
torch.cuda.synchronize()
print("ok", which)
if which.startswith("attnbwd"):
    T, nq, nkv, D = (4096, 32, 8, 128) if which == "attnbwd_tp1" else (4096, 4, 1, 128)
    qkv = (torch.randn(T, (nq + 2 * nkv) * D, device="cuda") * 0.5).to(torch.bfloat16)
    q, k_, v = qkv[:, :nq * D], qkv[:, nq * D:(nq + nkv) * D], qkv[:, (nq + nkv) * D:]
    o = torch.empty(T, nq * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    dh.attn_fwd(q, k_, v, o, lse, nq, nkv, D, D ** -0.5)
    do = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    for _ in range(2):
        dh.attn_bwd(q, k_, v, o, lse, do, dqkv[:, :nq * D], dqkv[:, nq * D:(nq + nkv) * D],
                    dqkv[:, (nq + nkv) * D:], nq, nkv, D, D ** -0.5)
    torch.cuda.synchronize()
    print("ok", which)
