"""The C-ABI libraries load without a GPU and export every function their
public headers declare (include/dh_capi.h -> libdh_b200.so, include/weft_capi.h
-> libweft_b200.so). No compute calls: this runs on the CPU-only builder."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2411_15871_b200", "lib")


def declared(header: str, prefix: str) -> list[str]:
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)  # drop comments
    text = re.sub(r"//[^\n]*", "", text)
    names = set(re.findall(r"\b(" + prefix + r"[A-Za-z0-9_]*)\s*\(", text))
    return sorted(names)


@pytest.mark.parametrize("header,lib,prefix", [("dh_capi.h", "libdh_b200.so", "dh_"),
                                               ("weft_capi.h", "libweft_b200.so", "weft_")])
def test_every_declared_symbol_is_exported(header, lib, prefix):
    path = os.path.join(LIB, lib)
    if not os.path.exists(path):
        pytest.skip(f"{lib} not built (run `make`)")
    names = declared(header, prefix)
    assert len(names) >= 9, names
    so = ctypes.CDLL(path)
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, f"{lib} lacks {missing}"


def test_planner_entry_points_reachable_without_gpu():
    from paper_2411_15871_b200.planner import lib
    r = lib().pipeline("w_shape", 4, 1)
    assert r["violations"] == [] and r["makespan_us"] > 0
