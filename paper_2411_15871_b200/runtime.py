"""Host-side Python mirror of the dh runtime C ABI (contexts, the TP+SP model,
SI plans, training steps). The runtime itself is C++/CUDA (csrc/runtime,
csrc/cuda); this module marshals arguments and exposes device buffers to
torch as zero-copy views. No fallback: a missing library or GPU raises.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass

from . import device as _dev
from .device import DeviceError, check

c_void_p, c_int, c_ll, c_float, c_char_p = (ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong,
                                            ctypes.c_float, ctypes.c_char_p)


class ModelCfg(ctypes.Structure):
    _fields_ = [("hidden", c_int), ("ffn", c_int), ("n_heads", c_int), ("n_kv_heads", c_int),
                ("head_dim", c_int), ("layers", c_int), ("seq_len", c_int),
                ("micro_batches", c_int), ("rope_theta", c_float), ("norm_eps", c_float),
                ("seed", ctypes.c_ulonglong), ("init_std", c_float),
                ("slots", c_int), ("split_layer", c_int), ("pp_rank", c_int), ("pp_size", c_int),
                ("experts", c_int), ("topk", c_int), ("capacity", c_int), ("context_parallel", c_int)]


class OptimCfg(ctypes.Structure):
    _fields_ = [("lr", c_float), ("beta1", c_float), ("beta2", c_float), ("eps", c_float),
                ("weight_decay", c_float), ("enabled", c_int)]


_SIGS = {
    "dh_ctx_create": ([c_int, c_int, c_int, c_void_p, c_int, ctypes.POINTER(c_void_p)], c_int),
    "dh_ctx_create_pp": ([c_int, c_int, c_int, c_void_p, c_int, c_int, c_void_p, c_int,
                          ctypes.POINTER(c_void_p)], c_int),
    "dh_loopback_group_create": ([c_int, c_int, ctypes.POINTER(c_void_p)], c_int),
    "dh_loopback_pp_group_create": ([c_int, c_int, ctypes.POINTER(c_void_p)], c_int),
    "dh_ctx_create_emulated": ([c_int, c_int, c_int, ctypes.c_double, ctypes.POINTER(c_void_p)], c_int),
    "dh_ctx_destroy": ([c_void_p], c_int),
    "dh_ctx_stream": ([c_void_p, c_int], c_void_p),
    "dh_comm_run": ([c_void_p, c_int, c_void_p, c_void_p, c_ll, c_int], c_int),
    "dh_nccl_unique_id": ([c_void_p], c_int),
    "dh_model_create": ([c_void_p, ctypes.POINTER(ModelCfg), ctypes.POINTER(c_void_p)], c_int),
    "dh_model_destroy": ([c_void_p], c_int),
    "dh_model_set_plan": ([c_void_p, c_char_p, c_char_p, c_char_p, c_int], c_int),
    "dh_model_set_overlap_ctas": ([c_void_p, c_int], c_int),
    "dh_model_set_fuse_optimizer": ([c_void_p, c_int], c_int),
    "dh_model_step": ([c_void_p, ctypes.POINTER(OptimCfg), c_int], c_int),
    "dh_model_run_program": ([c_void_p, c_int], c_int),
    "dh_model_zero_grads": ([c_void_p], c_int),
    "dh_model_sync": ([c_void_p], c_int),
    "dh_model_tensor": ([c_void_p, c_char_p, c_int, c_int, ctypes.POINTER(c_void_p),
                         ctypes.POINTER(c_ll), ctypes.POINTER(c_int)], c_int),
    "dh_model_info_json": ([c_void_p, ctypes.POINTER(c_void_p)], c_int),
    "dh_free_string": ([c_void_p], None),
    "dh_profile_json": ([c_void_p, c_int, ctypes.POINTER(c_void_p)], c_int),
    "dh_model_probe": ([c_void_p, c_int], c_int),
    "dh_model_set_skip_comm": ([c_void_p, c_int], c_int),
    "dh_lower_json": ([ctypes.POINTER(ModelCfg), c_int, c_int, c_char_p, c_char_p, c_int,
                       ctypes.POINTER(c_void_p)], c_int),
    "dh_model_probe_read": ([c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_int)], c_int),
    "dh_model_probe_read_node": ([c_void_p, c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_int)], c_int),
}
_bound = False


def _lib():
    global _bound
    lib = _dev.lib()
    if not _bound:
        for name, (args, res) in _SIGS.items():
            if hasattr(lib, name):
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
        _bound = True
    return lib


def _take_string(p: c_void_p) -> str:
    try:
        return ctypes.string_at(p.value).decode()
    finally:
        _lib().dh_free_string(p)


class _CudaArray:
    """__cuda_array_interface__ shim: a torch view of a pool buffer."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 2, "strides": None}


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(_lib().dh_nccl_unique_id(buf))
    return buf.raw


class Context:
    """One GPU / TP rank: lane streams + collective backend (include/dh_capi.h)."""

    def __init__(self, handle, tp_rank=0, tp_size=1):
        self.handle = handle
        self.tp_rank, self.tp_size = tp_rank, tp_size

    @classmethod
    def create(cls, device=0, tp_rank=0, tp_size=1, nccl_id: bytes | None = None, nccl_max_ctas=0):
        h = c_void_p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        check(_lib().dh_ctx_create(device, tp_rank, tp_size, idbuf, nccl_max_ctas, ctypes.byref(h)))
        return cls(h, tp_rank, tp_size)

    @classmethod
    def create_pp(cls, device=0, pp_rank=0, pp_size=2, pp_id: bytes | None = None, tp_rank=0, tp_size=1,
                  tp_id: bytes | None = None, nccl_max_ctas=0):
        """One W-pipeline stage on `device`: stage transfers over NCCL (dh_ctx_create_pp)."""
        h = c_void_p()
        buf = lambda b: ctypes.create_string_buffer(b, 128) if b else None  # noqa: E731
        check(_lib().dh_ctx_create_pp(device, tp_rank, tp_size, buf(tp_id), pp_rank, pp_size, buf(pp_id),
                                      nccl_max_ctas, ctypes.byref(h)))
        return cls(h, tp_rank, tp_size)

    @classmethod
    def loopback_pp_group(cls, device=0, pp_size=2):
        """pp_size pipeline-stage contexts on one device (staged-copy transfers)."""
        arr = (c_void_p * pp_size)()
        check(_lib().dh_loopback_pp_group_create(device, pp_size, arr))
        return [cls(c_void_p(arr[r]), 0, 1) for r in range(pp_size)]

    @classmethod
    def loopback_group(cls, device=0, tp_size=2):
        arr = (c_void_p * tp_size)()
        check(_lib().dh_loopback_group_create(device, tp_size, arr))
        return [cls(c_void_p(arr[r]), r, tp_size) for r in range(tp_size)]

    @classmethod
    def emulated(cls, device=0, tp_size=8, comm_ctas=16, link_gbs=770.0):
        """Per-rank shapes of a tp_size group on one GPU, collectives replaced by
        timing/SM-faithful proxy kernels (performance studies only)."""
        h = c_void_p()
        check(_lib().dh_ctx_create_emulated(device, tp_size, comm_ctas, link_gbs, ctypes.byref(h)))
        return cls(h, 0, tp_size)

    COMM_OPS = {"all_gather": 0, "reduce_scatter": 1, "all_reduce_f32": 2, "all_to_all": 3}

    def collective(self, op: str, send, recv, count: int, lane: int = 1):
        """Enqueue one collective of this context's group (dh_comm_run) on a lane
        stream; `send` / `recv` are CUDA tensors (bf16, fp32 for all_reduce_f32)."""
        check(_lib().dh_comm_run(self.handle, self.COMM_OPS[op], send.data_ptr(), recv.data_ptr(), count, lane))

    def stream_ptr(self, lane=0) -> int:
        return _lib().dh_ctx_stream(self.handle, lane)

    def close(self):
        if self.handle:
            check(_lib().dh_ctx_destroy(self.handle))
            self.handle = None


@dataclass
class LlamaShape:
    hidden: int
    ffn: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    layers: int
    seq_len: int
    micro_batches: int = 2
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    seed: int = 1234
    init_std: float = 0.02
    # pipeline stage (dh_model_cfg): 0 = single stage
    slots: int = 0
    split_layer: int = 0
    pp_rank: int = 0
    pp_size: int = 0
    # MoE (moe_ep template; 0 = dense): experts, top-k, slots per expert per
    # source rank (0 = ceil(1.25 * seq * topk / experts) rounded up to 32)
    experts: int = 0
    topk: int = 0
    capacity: int = 0
    # context parallelism: 1 = the context's group is the CP group (TP = 1)
    context_parallel: int = 0

    @property
    def moe(self) -> bool:
        return self.experts > 1

    def to_c(self) -> ModelCfg:
        return ModelCfg(self.hidden, self.ffn, self.n_heads, self.n_kv_heads, self.head_dim,
                        self.layers, self.seq_len, self.micro_batches, self.rope_theta,
                        self.norm_eps, self.seed, self.init_std, self.slots, self.split_layer,
                        self.pp_rank, self.pp_size, self.experts, self.topk, self.capacity,
                        self.context_parallel)

    def planner_model(self) -> dict:
        if self.moe:
            return {"name": "moe", "family": "phi_moe", "hidden": self.hidden,
                    "intermediate": self.ffn, "layers": self.layers, "seq_len": self.seq_len,
                    "experts": self.experts, "topk": self.topk or 2}
        return {"name": "llama", "family": "llama", "hidden": self.hidden,
                "intermediate": self.ffn, "layers": self.layers, "seq_len": self.seq_len}

    def moe_capacity(self) -> int:
        k = self.topk or 2
        c = -(-self.seq_len * k * 5 // (4 * self.experts))
        return self.capacity or (c + 31) // 32 * 32


LLAMA3_8B = LlamaShape(hidden=4096, ffn=14336, n_heads=32, n_kv_heads=8, head_dim=128, layers=32,
                       seq_len=4096, rope_theta=500000.0)
TINY = LlamaShape(hidden=256, ffn=768, n_heads=4, n_kv_heads=2, head_dim=64, layers=4, seq_len=128,
                  rope_theta=10000.0)
# BASELINE.json config 3 (GPT-3-13B-shaped: MHA, 40 x 128 heads; the dense_tp_sp
# template models every non-MoE family with a gated MLP, reference op_model.cpp:409)
GPT3_13B = LlamaShape(hidden=5120, ffn=20480, n_heads=40, n_kv_heads=40, head_dim=128, layers=40,
                      seq_len=2048, rope_theta=10000.0)
# BASELINE.json config 5 (Llama-2-70B-shaped, GQA 64 / 8 heads)
LLAMA2_70B = LlamaShape(hidden=8192, ffn=28672, n_heads=64, n_kv_heads=8, head_dim=128, layers=80,
                        seq_len=8192, rope_theta=10000.0)
# BASELINE.json config 4 (Phi-3.5-MoE-shaped: 16 experts top-2, expert ffn 6400,
# GQA 32 / 8 heads; seq 3072 as the reference's phi presets, presets.cpp phi-42B)
PHI35_MOE = LlamaShape(hidden=4096, ffn=6400, n_heads=32, n_kv_heads=8, head_dim=128, layers=32,
                       seq_len=3072, rope_theta=10000.0, experts=16, topk=2)
TINY_MOE = LlamaShape(hidden=256, ffn=512, n_heads=4, n_kv_heads=2, head_dim=64, layers=2, seq_len=128,
                      rope_theta=10000.0, experts=4, topk=2)


class Model:
    """The Llama TP+SP layer stack on one rank (csrc/runtime/model.cpp)."""

    def __init__(self, ctx: Context, shape: LlamaShape):
        self.ctx, self.shape = ctx, shape
        self.handle = c_void_p()
        cfg = shape.to_c()
        check(_lib().dh_model_create(ctx.handle, ctypes.byref(cfg), ctypes.byref(self.handle)))

    def set_plan(self, plan_json: str | None = None, profile_json: str | None = None,
                 cluster_json: str | None = None, mode: str = "si"):
        enc = lambda s: None if s is None else s.encode()  # noqa: E731
        check(_lib().dh_model_set_plan(self.handle, enc(plan_json), enc(profile_json),
                                       enc(cluster_json), {"si": 0, "sequential": 1, "si_relaxed": 2,
                                                             "w_pipeline": 3, "si_deferred": 4}[mode]))

    def set_fuse_optimizer(self, on: bool):
        """Per-layer AdamW inside the program (default); effective at the next set_plan."""
        check(_lib().dh_model_set_fuse_optimizer(self.handle, int(on)))

    def set_overlap_ctas(self, n: int):
        check(_lib().dh_model_set_overlap_ctas(self.handle, n))

    def step(self, optim: dict | None = None, use_graph=True):
        oc = None
        if optim is not None:
            oc = OptimCfg(optim.get("lr", 1e-4), optim.get("beta1", 0.9), optim.get("beta2", 0.95),
                          optim.get("eps", 1e-8), optim.get("weight_decay", 0.0), 1)
        check(_lib().dh_model_step(self.handle, ctypes.byref(oc) if oc else None, int(use_graph)))

    def run_program(self, use_graph=False):
        check(_lib().dh_model_run_program(self.handle, int(use_graph)))

    def zero_grads(self):
        check(_lib().dh_model_zero_grads(self.handle))

    def sync(self):
        check(_lib().dh_model_sync(self.handle))

    def tensor(self, name: str, layer: int = 0, strand: int = 0):
        import torch
        p, n, dt = c_void_p(), c_ll(), c_int()
        check(_lib().dh_model_tensor(self.handle, name.encode(), layer, strand, ctypes.byref(p),
                                     ctypes.byref(n), ctypes.byref(dt)))
        if dt.value == 1:
            return torch.as_tensor(_CudaArray(p.value, (n.value,), "<f4"), device="cuda")
        raw = torch.as_tensor(_CudaArray(p.value, (n.value,), "<i2"), device="cuda")
        return raw.view(torch.bfloat16)

    def info(self) -> dict:
        p = c_void_p()
        check(_lib().dh_model_info_json(self.handle, ctypes.byref(p)))
        return json.loads(_take_string(p))

    def probe(self, node: int):
        """Also time every launch of template node `node` (-1 clears all probes)."""
        check(_lib().dh_model_probe(self.handle, node))

    def set_skip_comm(self, skip: bool):
        check(_lib().dh_model_set_skip_comm(self.handle, int(skip)))

    def probe_read(self, node: int = -1):
        """(summed ms, launches) of probed node `node` (-1: the first probed)."""
        ms, n = ctypes.c_double(), c_int()
        check(_lib().dh_model_probe_read_node(self.handle, node, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def profile(self, iters=10) -> str:
        p = c_void_p()
        check(_lib().dh_profile_json(self.handle, iters, ctypes.byref(p)))
        return _take_string(p)

    def close(self):
        if self.handle:
            check(_lib().dh_model_destroy(self.handle))
            self.handle = None


def lower(shape: "LlamaShape", tp: int, plan_json: str | None, mode: str = "si", rank: int = 0,
          profile_json: str | None = None) -> dict:
    """Host-only lowering of a plan to the executor's launch program (no GPU)."""
    cfg = shape.to_c()
    p = c_void_p()
    enc = lambda s: None if s is None else s.encode()  # noqa: E731
    check(_lib().dh_lower_json(ctypes.byref(cfg), tp, rank, enc(plan_json), enc(profile_json),
                               {"si": 0, "sequential": 1, "si_relaxed": 2, "w_pipeline": 3, "si_deferred": 4}[mode],
                               ctypes.byref(p)))
    return json.loads(_take_string(p))


__all__ = ["lower", "Context", "Model", "LlamaShape", "LLAMA3_8B", "TINY", "PHI35_MOE", "TINY_MOE",
           "DeviceError", "nccl_unique_id"]
