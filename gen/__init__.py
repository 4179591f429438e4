"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

Holds none of the hot path's arithmetic (see gen/problem.py and gen/dip_gen.c
headers). The C candidate generator is compiled in-tree with gcc on first use
(or by `__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

from .problem import (CONFIG_NAMES, Module, Problem, make_problem, problem_arrays,  # noqa: F401
                      splitmix64, substream)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libdipgen.so")
_SRC = os.path.join(_HERE, "dip_gen.c")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", _SO, _SRC])
    return _SO


class _GenCfg(ctypes.Structure):
    _fields_ = [
        ("P", ctypes.c_uint32), ("nmod", ctypes.c_uint32), ("m", ctypes.c_uint32),
        ("n_max", ctypes.c_uint32), ("fbw", ctypes.c_uint32),
        ("K", ctypes.c_void_p), ("max_split", ctypes.c_void_p), ("producer_mask", ctypes.c_void_p),
        ("nbi", ctypes.c_void_p), ("seed", ctypes.c_uint64), ("mode", ctypes.c_uint32),
        ("split_rule_b", ctypes.c_uint32), ("p_mutate", ctypes.c_double), ("p_bad", ctypes.c_double),
    ]


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        _lib.dip_gen_candidates.restype = ctypes.c_int
        _lib.dip_gen_candidates.argtypes = [ctypes.POINTER(_GenCfg), ctypes.c_uint64, ctypes.c_uint64] + \
            [ctypes.c_void_p] * 6 + [ctypes.c_int]
    return _lib


class Candidates:
    """Host view of a candidate batch (SoA), the layout `dip_encode_candidates` reads."""

    def __init__(self, pb: Problem, count: int):
        self.count = count
        self.split = np.zeros((count, pb.m * pb.nmod), np.uint8)
        self.n = np.zeros(count, np.uint32)
        self.fwd = np.full((count, pb.n_max), 0xFFFF, np.uint16)
        self.bwd = np.full((count, pb.n_max), 0xFFFF, np.uint16)
        self.fb = np.zeros((count, pb.P, pb.fbw), np.uint32)
        self.family = np.zeros(count, np.uint8)

    def subset(self, idx) -> "Candidates":
        c = Candidates.__new__(Candidates)
        idx = np.asarray(idx)
        c.count = len(idx)
        for k in ("split", "n", "fwd", "bwd", "fb", "family"):
            setattr(c, k, np.ascontiguousarray(getattr(self, k)[idx]))
        return c


def generate(pb: Problem, first: int, count: int, mode: int = 0, seed: Optional[int] = None,
             threads: int = 0, p_mutate: float = 0.04, p_bad: float = 0.005,
             split_rule_b: int = 12) -> Candidates:
    """Candidates [first, first+count) of problem `pb` (pure function of (seed, index))."""
    lib = _load()
    c = Candidates(pb, count)
    if count == 0:
        return c
    arr = problem_arrays(pb)
    nbi = np.ascontiguousarray(pb.n_inst().reshape(-1).astype(np.uint32))
    if seed is None:
        seed = substream(pb.seed, "cands")
    cfg = _GenCfg(pb.P, pb.nmod, pb.m, pb.n_max, pb.fbw,
                  arr["K"].ctypes.data, arr["max_split"].ctypes.data, arr["producer_mask"].ctypes.data,
                  nbi.ctypes.data, seed & ((1 << 64) - 1), mode, split_rule_b, p_mutate, p_bad)
    if threads <= 0:
        threads = min(os.cpu_count() or 1, max(1, count // 64))
    rc = lib.dip_gen_candidates(ctypes.byref(cfg), first, count, c.split.ctypes.data, c.n.ctypes.data,
                                c.fwd.ctypes.data, c.bwd.ctypes.data, c.fb.ctypes.data,
                                c.family.ctypes.data, threads)
    if rc != 0:
        raise RuntimeError("candidate generator failed to complete an order")
    return c
