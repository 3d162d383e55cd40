"""Python mirror of the weft plan-time API over the C ABI (include/weft_capi.h).

The planner itself is host C++ (paper_2411_15871_b200/csrc/planner/, a bit-exact
re-implementation of /root/reference/proj/src/{op_model,overlap_profile,
pairing_search}.cpp); this module only marshals JSON across ctypes so tests,
the profiler driver and the executor can call it. Function names follow the
reference API:

    build_layer_dag          op_model.hpp:66-68
    enumerate_topological_orders  op_model.hpp:76
    segment_pair_cost        overlap_profile.hpp:72-73
    dp_align / brute_force_align  pairing_search.hpp:55,63
    search_si_plan + plan_to_json pairing_search.hpp:93-98

Errors are raised as the reference's exception classes (ConfigError etc.).
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Any

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libweft_b200.so")


class WeftError(RuntimeError):
    """weft::Error"""


class ConfigError(WeftError):
    """weft::ConfigError (CLI exit 2)"""


class InfeasibleError(WeftError):
    """weft::InfeasibleError (CLI exit 3)"""


class MissingProfileEntry(WeftError):
    """weft::MissingProfileEntry (CLI exit 4)"""


_STATUS = {2: ConfigError, 3: InfeasibleError, 4: MissingProfileEntry}

_FUNCS = ("build_dag_json", "topo_orders_json", "segment_cost_json", "dp_align_json",
          "search_json", "profile_roundtrip_json", "templates_json", "pipeline_json", "memory_json",
          "estimate_json")


class PlannerLib:
    """ctypes binding of one planner build; `prefix` selects weft_ or weft_ref_."""

    def __init__(self, path: str, prefix: str = "weft_"):
        if not os.path.exists(path):
            raise FileNotFoundError(f"planner library not built: {path} (run `make planner`)")
        self.path = path
        self._lib = ctypes.CDLL(path)
        self._prefix = prefix
        for f in _FUNCS:
            fn = getattr(self._lib, prefix + f)
            fn.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
            fn.restype = ctypes.c_int
        self._err = getattr(self._lib, prefix + "last_error")
        self._err.restype = ctypes.c_char_p
        self._free = getattr(self._lib, prefix + "free")
        self._free.argtypes = [ctypes.c_void_p]

    def call(self, name: str, request: dict[str, Any]) -> dict[str, Any]:
        out = ctypes.c_void_p()
        rc = getattr(self._lib, self._prefix + name)(json.dumps(request).encode(), ctypes.byref(out))
        if rc != 0:
            msg = self._err().decode()
            raise _STATUS.get(rc, WeftError)(msg)
        try:
            text = ctypes.string_at(out.value).decode()
        finally:
            self._free(out)
        return json.loads(text)

    # --- reference-named entry points -----------------------------------------
    def build_layer_dag(self, model, parallelism, cluster, profile=None, use_profile_solo=True):
        req = {"model": model, "parallelism": parallelism, "cluster": cluster,
               "use_profile_solo": use_profile_solo}
        if profile is not None:
            req["profile"] = profile
        r = self.call("build_dag_json", req)
        return r["fwd"], r["bwd"]

    def enumerate_topological_orders(self, dag=None, cap=16, **scenario):
        req = dict(scenario, cap=cap)
        if dag is not None:
            req["dag"] = dag
        return self.call("topo_orders_json", req)["orders"]

    def segment_pair_cost(self, seg_a, seg_b, profile):
        return self.call("segment_cost_json", {"a": seg_a, "b": seg_b, "profile": profile})

    def dp_align(self, cost, barrier_cost_us=0.0, brute_force=False):
        n_f, n_b = len(cost) - 1, len(cost[0]) - 1
        return self.call("dp_align_json", {"n_f": n_f, "n_b": n_b, "cost": cost,
                                           "barrier_cost_us": barrier_cost_us,
                                           "brute_force": brute_force})

    def search_si_plan(self, model, parallelism, cluster, profile, caps=None,
                       barrier_cost_us=0.0, parallel=False, threads=0, metadata=None, repeat=1):
        req = {"model": model, "parallelism": parallelism, "cluster": cluster,
               "profile": profile, "barrier_cost_us": barrier_cost_us, "parallel": parallel,
               "threads": threads, "repeat": repeat}
        if caps:
            req["caps"] = caps
        if metadata:
            req["metadata"] = metadata
        return self.call("search_json", req)

    def profile_to_json(self, profile):
        return self.call("profile_roundtrip_json", {"profile": profile})["profile_json"]

    def builtin_template_json(self):
        return self.call("templates_json", {})["builtin_template_json"]

    def pipeline(self, discipline, m, p, f_us=1.0, b_us=1.0, si_us=2.0, fold_layers=None):
        """schedule_{w_pipeline,1f1b,bidirectional} + analyses (folding_pipeline.hpp)."""
        req = {"schedule": {"discipline": discipline, "m": m, "p": p, "f_us": f_us, "b_us": b_us,
                            "si_us": si_us}}
        if fold_layers is not None:
            req["fold_layers"] = fold_layers
        return self.call("pipeline_json", req)

    def memory(self, memory, schedule=None, model=None, parallelism=None, max_model=None):
        """simulate_memory / max_model_size / default footprints (memory_sim.hpp)."""
        req = {"memory": memory}
        for k, v in (("schedule", schedule), ("model", model), ("parallelism", parallelism),
                     ("max_model", max_model)):
            if v is not None:
                req[k] = v
        return self.call("memory_json", req)

    def estimate(self, model, parallelism, cluster, profile, source="dhelix", microbatches=8, caps=None):
        """estimate_iteration_time (estimate.hpp)."""
        req = {"model": model, "parallelism": parallelism, "cluster": cluster, "profile": profile,
               "source": source, "microbatches": microbatches}
        if caps:
            req["caps"] = caps
        return self.call("estimate_json", req)

    def compare(self, scenario: dict):
        """compare_report on a scenario document (report.hpp): one row per plan source."""
        r = self.call("compare_json", {"scenario": scenario})
        r["report"] = json.loads(r["report_json"])
        return r

    def comm_volume(self, model, parallelism, cluster, tokens, microbatches=1):
        """comm_volume_estimate (comm_volume.hpp)."""
        return self.call("comm_volume_json", {"model": model, "parallelism": parallelism, "cluster": cluster,
                                              "tokens": tokens, "microbatches": microbatches})


_default: PlannerLib | None = None


def lib() -> PlannerLib:
    global _default
    if _default is None:
        _default = PlannerLib(LIB_PATH, "weft_")
    return _default


def parse_plan(plan_json: str) -> dict[str, Any]:
    """Parse an SI-plan document (the plan_to_json schema,
    /root/reference/proj/src/pairing_search.cpp:543-561) and validate it."""
    p = json.loads(plan_json)
    for key in ("steps", "fwd_seq", "bwd_seq", "fwd_cuts", "bwd_cuts", "total_us"):
        if key not in p:
            raise ConfigError(f"plan schema error: missing '{key}'")

    def segs(seq, cuts):
        bounds = [0] + list(cuts) + [len(seq)]
        if any(b >= a for a, b in zip(bounds[1:], bounds[:-1])):
            raise ConfigError("segmentation cuts must be strictly increasing within (0, len)")
        return [seq[bounds[k]:bounds[k + 1]] for k in range(len(bounds) - 1)] if seq else []

    p["fwd_segments"] = segs(p["fwd_seq"], p["fwd_cuts"])
    p["bwd_segments"] = segs(p["bwd_seq"], p["bwd_cuts"])
    nf, nb = 1, 1
    for st in p["steps"]:
        f, b = st["fwd_seg"], st["bwd_seg"]
        if f is None and b is None:
            raise ConfigError("plan step with neither segment")
        if f is not None:
            if f != nf:
                raise ConfigError("plan steps not monotone in fwd segments")
            nf += 1
        if b is not None:
            if b != nb:
                raise ConfigError("plan steps not monotone in bwd segments")
            nb += 1
    if nf != len(p["fwd_segments"]) + 1 or nb != len(p["bwd_segments"]) + 1:
        raise ConfigError("plan steps do not cover every segment")
    return p
