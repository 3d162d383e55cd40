"""ctypes binding of the dh C ABI (include/dh_capi.h) -> libdh_b200.so.

torch is used only for device memory and streams: tensors are passed to the
native kernels as raw pointers. There is no fallback path: if the CUDA
library is missing or no GPU is present, every call raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DH_LIB_PATH: load an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("DH_LIB_PATH") or os.path.join(_HERE, "lib", "libdh_b200.so")

_lib = None


class DeviceError(RuntimeError):
    """dh status != DH_OK (maps to weft::DeviceError on the C++ side)."""


c_void_p, c_int, c_ll, c_float, c_ull = (ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong,
                                         ctypes.c_float, ctypes.c_ulonglong)


class GemmArgs(ctypes.Structure):
    _fields_ = [("a", c_void_p), ("lda", c_ll), ("a_mn", c_int),
                ("b", c_void_p), ("ldb", c_ll), ("b_mn", c_int),
                ("d", c_void_p), ("ldd", c_ll), ("d_fp32", c_int),
                ("m", c_int), ("n", c_int), ("k", c_int),
                ("accumulate", c_int), ("max_ctas", c_int), ("tile_n", c_int),
                ("epilogue", c_int), ("d2", c_void_p), ("aux0", c_void_p), ("aux1", c_void_p),
                ("ld_aux", c_ll), ("a2", c_void_p), ("lda2", c_ll), ("b2", c_void_p), ("ldb2", c_ll),
                ("k2", c_int), ("d_m2", c_void_p), ("ldd_m2", c_ll), ("m2", c_int)]


EPI_NONE, EPI_SWIGLU_FWD, EPI_SWIGLU_FWD_UP, EPI_SWIGLU_BWD, EPI_SWIGLU_PAIR = 0, 1, 2, 3, 4


_SIGS = {
    "dh_gemm": [ctypes.POINTER(GemmArgs), c_void_p],
    "dh_rmsnorm_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_float, c_void_p],
    "dh_add_rmsnorm_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_float,
                           c_void_p],
    "dh_rmsnorm_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                       c_void_p, c_int, c_int, c_void_p],
    "dh_add": [c_void_p, c_void_p, c_void_p, c_ll, c_void_p],
    "dh_swiglu_fwd": [c_void_p, c_void_p, c_void_p, c_ll, c_void_p],
    "dh_swiglu_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_ll, c_void_p],
    "dh_rope": [c_void_p, c_ll, c_int, c_int, c_int, c_int, c_float, c_int, c_int, c_void_p],
    "dh_attn_fwd_scratch_floats": [c_int, c_int, c_int, c_int],
    "dh_attn_fwd": [c_void_p, c_void_p, c_void_p, c_ll, c_ll, c_void_p, c_ll, c_void_p, c_void_p,
                    c_ll, c_int, c_int, c_int, c_int, c_float, c_void_p],
    "dh_attn_bwd": [c_void_p, c_void_p, c_void_p, c_ll, c_ll, c_void_p, c_ll, c_void_p, c_void_p,
                    c_void_p, c_void_p, c_void_p, c_ll, c_ll, c_void_p, c_int, c_int, c_int,
                    c_int, c_float, c_void_p],
    "dh_attn_fwd_scratch_floats_ex": [c_int, c_int, c_int, c_int, c_int, c_int],
    "dh_attn_bwd_scratch_floats": [c_int, c_int, c_int, c_int],
    "dh_attn_bwd_scratch_floats_ex": [c_int, c_int, c_int, c_int, c_int, c_int],
    "dh_attn_fwd_ex": [c_void_p, c_void_p, c_void_p, c_ll, c_ll, c_void_p, c_ll, c_void_p, c_void_p,
                       c_ll, c_int, c_int, c_int, c_int, c_int, c_int, c_float, c_void_p],
    "dh_attn_bwd_ex": [c_void_p, c_void_p, c_void_p, c_ll, c_ll, c_void_p, c_ll, c_void_p, c_void_p,
                       c_void_p, c_void_p, c_void_p, c_ll, c_ll, c_void_p, c_int, c_int, c_int, c_int, c_int,
                       c_int, c_float, c_void_p],
    "dh_adamw": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_ll, c_float, c_float,
                 c_float, c_float, c_float, c_int, c_float, c_int, c_void_p],
    "dh_init_normal": [c_void_p, c_void_p, c_ll, c_ull, c_float, c_void_p],
    "dh_fill_bf16": [c_void_p, c_float, c_ll, c_void_p],
    "dh_moe_router_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p],
    "dh_moe_assign": [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p],
    "dh_moe_permute": [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p],
    "dh_moe_unpermute": [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p],
    "dh_moe_unpermute_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                             c_void_p],
    "dh_moe_permute_bwd": [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p],
    "dh_moe_router_bwd_scratch_floats": [c_int, c_int, c_int],
    "dh_moe_router_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                          c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p],
}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"CUDA library not built: {LIB_PATH} (run `make cuda`)")
        # torch bundles a newer libnccl.so.2 than the system one we link; load
        # torch first so both resolve the soname to torch's copy (loading ours
        # first would bind the older system NCCL and break `import torch`).
        import torch  # noqa: F401
        l = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, args in _SIGS.items():
            if not hasattr(l, name):
                continue  # symbol not built yet: calling it raises AttributeError
            fn = getattr(l, name)
            fn.argtypes = args
            fn.restype = c_int
        l.dh_last_error.restype = ctypes.c_char_p
        l.dh_attn_fwd_scratch_floats.restype = c_ll
        l.dh_attn_fwd_scratch_floats_ex.restype = c_ll
        l.dh_attn_bwd_scratch_floats.restype = c_ll
        l.dh_attn_bwd_scratch_floats_ex.restype = c_ll
        if hasattr(l, "dh_moe_router_bwd_scratch_floats"):
            l.dh_moe_router_bwd_scratch_floats.restype = c_ll
        _lib = l
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise DeviceError(f"dh status {rc}: {lib().dh_last_error().decode()}")


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# --------------------------------------------------------------------------- kernels

def gemm(a, b, d, *, a_mn=False, b_mn=False, accumulate=False, m=None, n=None, k=None,
         max_ctas=0, tile_n=0, stream=None, epilogue=EPI_NONE, d2=None, aux0=None, aux1=None,
         a2=None, b2=None, k2=0, d_m2=None, m2=0):
    """d(m,n) (+)= sum_k A(m,k) B(n,k). A = a[m,k] (K-major) or a[k,m] (a_mn);
    B = b[n,k] (K-major) or b[k,n] (b_mn). d bf16 or fp32 [m,n].
    epilogue = EPI_SWIGLU_*: fused SwiGLU (see dh_capi.h) writing d and d2 from aux0/aux1.
    Two segments in one launch: k2 > 0 adds a2 @ b2^T (K-concatenation); m2 > 0 computes a2's
    rows (m2 of them) into d_m2 (M-concatenation)."""
    import torch
    if m is None:
        m = a.shape[1] if a_mn else a.shape[0]
    if k is None:
        k = a.shape[0] if a_mn else a.shape[1]
    if n is None:
        n = b.shape[1] if b_mn else b.shape[0]
    args = GemmArgs(a.data_ptr(), a.stride(0), int(a_mn), b.data_ptr(), b.stride(0), int(b_mn),
                    d.data_ptr(), d.stride(0), int(d.dtype == torch.float32), m, n, k,
                    int(accumulate), max_ctas, tile_n, epilogue, _ptr(d2), _ptr(aux0), _ptr(aux1),
                    d.stride(0))
    if a2 is not None:
        args.a2, args.lda2 = a2.data_ptr(), a2.stride(0)
    if b2 is not None:
        args.b2, args.ldb2 = b2.data_ptr(), b2.stride(0)
    if d_m2 is not None:
        args.d_m2, args.ldd_m2 = d_m2.data_ptr(), d_m2.stride(0)
    args.k2, args.m2 = k2, m2
    check(lib().dh_gemm(ctypes.byref(args), _stream(stream)))
    return d


def rmsnorm_fwd(x, gamma, y, rstd, eps=1e-5, stream=None):
    rows, cols = x.shape
    check(lib().dh_rmsnorm_fwd(_ptr(x), _ptr(gamma), _ptr(y), _ptr(rstd), rows, cols, eps,
                               _stream(stream)))


def add_rmsnorm_fwd(x, resid, x_out, gamma, y, rstd, eps=1e-5, stream=None):
    """x_out = bf16(x + resid); y = RMSNorm(x_out) (the fused bda0 + ln1 node)."""
    rows, cols = x.shape
    check(lib().dh_add_rmsnorm_fwd(_ptr(x), _ptr(resid), _ptr(x_out), _ptr(gamma), _ptr(y), _ptr(rstd), rows, cols,
                                   eps, _stream(stream)))


def rmsnorm_bwd(x, gamma, rstd, dy, dx, dgamma_acc=None, partial=None, resid=None, stream=None):
    import torch
    rows, cols = x.shape
    if partial is None:
        partial = torch.empty(min(rows, 1184) * cols, dtype=torch.float32, device=x.device)
    check(lib().dh_rmsnorm_bwd(_ptr(x), _ptr(gamma), _ptr(rstd), _ptr(dy), _ptr(resid), _ptr(dx),
                               _ptr(dgamma_acc), _ptr(partial), rows, cols, _stream(stream)))


def add(a, b, out, stream=None):
    check(lib().dh_add(_ptr(a), _ptr(b), _ptr(out), a.numel(), _stream(stream)))


def swiglu_fwd(gate, up, act, stream=None):
    check(lib().dh_swiglu_fwd(_ptr(gate), _ptr(up), _ptr(act), gate.numel(), _stream(stream)))


def swiglu_bwd(gate, up, dact, dgate, dup, stream=None):
    check(lib().dh_swiglu_bwd(_ptr(gate), _ptr(up), _ptr(dact), _ptr(dgate), _ptr(dup),
                              gate.numel(), _stream(stream)))


def rope(qkv, n_q_heads, n_kv_heads, head_dim, theta, pos0=0, inverse=False, tokens=None,
         stream=None):
    tokens = qkv.shape[0] if tokens is None else tokens
    check(lib().dh_rope(_ptr(qkv), qkv.stride(0), tokens, n_q_heads, n_kv_heads, head_dim, theta,
                        pos0, int(inverse), _stream(stream)))


def attn_fwd_scratch_floats(tokens, n_q_heads, n_kv_heads, head_dim):
    return int(lib().dh_attn_fwd_scratch_floats(tokens, n_q_heads, n_kv_heads, head_dim))


def attn_fwd(q, k, v, o, lse, n_q_heads, n_kv_heads, head_dim, scale, stream=None, split=True):
    """split=True allocates the KV-split scratch when the launcher wants it."""
    import torch
    tokens = q.shape[0]
    n = attn_fwd_scratch_floats(tokens, n_q_heads, n_kv_heads, head_dim) if split else 0
    scratch = torch.empty(max(n, 1), dtype=torch.float32, device=q.device) if n else None
    check(lib().dh_attn_fwd(_ptr(q), _ptr(k), _ptr(v), q.stride(0), k.stride(0), _ptr(o),
                            o.stride(0), _ptr(lse), _ptr(scratch) if n else None, n, tokens,
                            n_q_heads, n_kv_heads, head_dim, scale, _stream(stream)))


def attn_bwd_scratch_floats(tokens, n_q_heads, n_kv_heads, head_dim, tokens_kv=None, q_offset=0):
    """fp32 scratch of the attention backward (its work plan's partial slots)."""
    return int(lib().dh_attn_bwd_scratch_floats_ex(tokens, n_q_heads, n_kv_heads, head_dim,
                                                   tokens if tokens_kv is None else tokens_kv, q_offset))


def attn_bwd(q, k, v, o, lse, do, dq, dk, dv, n_q_heads, n_kv_heads, head_dim, scale,
             scratch=None, stream=None):
    import torch
    tokens = q.shape[0]
    need = attn_bwd_scratch_floats(tokens, n_q_heads, n_kv_heads, head_dim)
    if scratch is None:
        scratch = torch.empty(need, dtype=torch.float32, device=q.device)
    elif scratch.numel() < need:
        raise DeviceError(f"attn_bwd: scratch has {scratch.numel()} floats, needs {need}")
    check(lib().dh_attn_bwd(_ptr(q), _ptr(k), _ptr(v), q.stride(0), k.stride(0), _ptr(o),
                            o.stride(0), _ptr(lse), _ptr(do), _ptr(dq), _ptr(dk), _ptr(dv),
                            dq.stride(0), dk.stride(0), _ptr(scratch), tokens, n_q_heads,
                            n_kv_heads, head_dim, scale, _stream(stream)))


def attn_fwd_cp(q, k, v, o, lse, q_offset, n_q_heads, n_kv_heads, head_dim, scale, stream=None):
    """Context-parallel forward: q rows at global positions [q_offset, q_offset + len(q))
    against every key row of k / v (causal)."""
    import torch
    tq, tk = q.shape[0], k.shape[0]
    n = int(lib().dh_attn_fwd_scratch_floats_ex(tq, n_q_heads, n_kv_heads, head_dim, tk, q_offset))
    scratch = torch.empty(max(n, 1), dtype=torch.float32, device=q.device) if n else None
    check(lib().dh_attn_fwd_ex(_ptr(q), _ptr(k), _ptr(v), q.stride(0), k.stride(0), _ptr(o), o.stride(0),
                               _ptr(lse), _ptr(scratch) if n else None, n, tq, tk, q_offset, n_q_heads,
                               n_kv_heads, head_dim, scale, _stream(stream)))


def attn_bwd_cp(q, k, v, o, lse, do, dq, dk, dv, q_offset, n_q_heads, n_kv_heads, head_dim, scale, stream=None):
    """Context-parallel backward: dq for the local rows, dk / dv for every key row
    (the gradient from these queries only)."""
    import torch
    tq, tk = q.shape[0], k.shape[0]
    scratch = torch.empty(attn_bwd_scratch_floats(tq, n_q_heads, n_kv_heads, head_dim, tk, q_offset),
                          dtype=torch.float32, device=q.device)
    check(lib().dh_attn_bwd_ex(_ptr(q), _ptr(k), _ptr(v), q.stride(0), k.stride(0), _ptr(o), o.stride(0),
                               _ptr(lse), _ptr(do), _ptr(dq), _ptr(dk), _ptr(dv), dq.stride(0), dk.stride(0),
                               _ptr(scratch), tq, tk, q_offset, n_q_heads, n_kv_heads, head_dim, scale,
                               _stream(stream)))


def adamw(master, weight, grad, m, v, lr, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0, step=1,
          grad_scale=1.0, zero_grad=True, stream=None):
    """AdamW on fp32 master weights (in place); refreshes the bf16 `weight`."""
    check(lib().dh_adamw(_ptr(master), _ptr(weight), _ptr(grad), _ptr(m), _ptr(v), master.numel(), lr,
                         beta1, beta2, eps, weight_decay, step, grad_scale, int(zero_grad),
                         _stream(stream)))


# --------------------------------------------------------------------------- MoE (moe.cu)

def moe_router_fwd(x, wr, probs, ids, wts, topk, stream=None):
    """probs [T,E] f32 = softmax(x wr^T); ids int32 / wts f32 [T,K] = top-k."""
    T, H = x.shape
    check(lib().dh_moe_router_fwd(_ptr(x), _ptr(wr), _ptr(probs), _ptr(ids), _ptr(wts), T, H, wr.shape[0], topk,
                                  _stream(stream)))


def moe_assign(ids, experts, capacity, slot, slot_src, stream=None):
    T, K = ids.shape
    check(lib().dh_moe_assign(_ptr(ids), T, K, experts, capacity, _ptr(slot), _ptr(slot_src), _stream(stream)))


def moe_permute(x, slot_src, xp, topk, stream=None):
    check(lib().dh_moe_permute(_ptr(x), _ptr(slot_src), _ptr(xp), xp.shape[0], topk, x.shape[1], _stream(stream)))


def moe_unpermute(y, slot, wts, out, stream=None):
    T, K = slot.shape
    check(lib().dh_moe_unpermute(_ptr(y), _ptr(slot), _ptr(wts), _ptr(out), T, K, out.shape[1], _stream(stream)))


def moe_unpermute_bwd(dy, y, slot_src, wts, dys, dw, topk, stream=None):
    check(lib().dh_moe_unpermute_bwd(_ptr(dy), _ptr(y), _ptr(slot_src), _ptr(wts), _ptr(dys), _ptr(dw),
                                     y.shape[0], topk, y.shape[1], _stream(stream)))


def moe_permute_bwd(dxp, slot, dx, stream=None):
    T, K = slot.shape
    check(lib().dh_moe_permute_bwd(_ptr(dxp), _ptr(slot), _ptr(dx), T, K, dx.shape[1], _stream(stream)))


def moe_router_bwd(probs, ids, slot, dw, x, wr, dx_in, dx_out, dwr, stream=None):
    import torch
    T, H = x.shape
    E, K = wr.shape[0], ids.shape[1]
    n = int(lib().dh_moe_router_bwd_scratch_floats(T, H, E))
    scratch = torch.empty(n, dtype=torch.float32, device=x.device)
    check(lib().dh_moe_router_bwd(_ptr(probs), _ptr(ids), _ptr(slot), _ptr(dw), _ptr(x), _ptr(wr), _ptr(dx_in),
                                  _ptr(dx_out), _ptr(dwr), _ptr(scratch), T, H, E, K, _stream(stream)))
