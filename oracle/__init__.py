"""CPU oracle for DIP candidate-schedule scoring -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. It shares no code with the CUDA path
(paper_2504_14145_b200/) and never imports it; both read the same seeded
inputs from gen/ (data only).

The arithmetic lives in oracle/dip_oracle.c (plain C, O1-O11 of SURVEY.md
§8(c), each step citing the PAPER.md passage it follows). This wrapper only
marshals numpy arrays. Every function is pinned by tests/test_oracle_*.py
(see DESIGN.md §4 for the pin of each step).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dip_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

ST_OK, ST_OOM, ST_DEADLOCK, ST_BAD = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle with plain -O2 (no SIMD tricks: it is the slow reference)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", _SO, _SRC, "-lm"])
    return _SO


class _OProblem(ctypes.Structure):
    _fields_ = [("P", ctypes.c_uint32), ("nmod", ctypes.c_uint32), ("m", ctypes.c_uint32)] + \
        [(k, ctypes.c_void_p) for k in ("L", "K", "max_split", "w_max", "producer_mask", "tab_off",
                                        "tab_f", "tab_b", "tab_act", "tab_p2p", "chunk_off",
                                        "chunk_layers", "inst_off", "inst_units", "budget_kib")]


class _OCands(ctypes.Structure):
    _fields_ = [("n_max", ctypes.c_uint32), ("fbw", ctypes.c_uint32)] + \
        [(k, ctypes.c_void_p) for k in ("split", "n", "fwd", "bwd", "fb", "ord")]


def _load():
    global _lib
    if _lib is None:
        path = os.environ.get("ORACLE_LIB")        # e.g. a sanitizer build (tests/test_sanitizers.py)
        if not path:
            build()
            path = _SO
        lib = ctypes.CDLL(path)
        lib.oracle_chunk_layers.restype = ctypes.c_int
        lib.oracle_chunk_layers.argtypes = [ctypes.c_uint32] * 3 + [ctypes.c_void_p]
        lib.oracle_split.restype = ctypes.c_int
        lib.oracle_split.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p]
        lib.oracle_eval.restype = ctypes.c_int
        lib.oracle_eval.argtypes = [ctypes.POINTER(_OProblem), ctypes.POINTER(_OCands), ctypes.c_uint64,
                                    ctypes.c_uint64] + [ctypes.c_void_p] * 6 + [ctypes.c_int]
        lib.oracle_timeline.restype = ctypes.c_int
        lib.oracle_timeline.argtypes = [ctypes.POINTER(_OProblem), ctypes.POINTER(_OCands), ctypes.c_uint64,
                                        ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_interleave.restype = ctypes.c_int
        lib.oracle_interleave.argtypes = [ctypes.POINTER(_OProblem), ctypes.POINTER(_OCands), ctypes.c_uint64,
                                          ctypes.c_uint64] + [ctypes.c_void_p] * 7 + [ctypes.c_int]
        lib.oracle_search.restype = ctypes.c_int
        lib.oracle_search.argtypes = [ctypes.POINTER(_OProblem), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                                      ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_double, ctypes.c_double] + [ctypes.c_void_p] * 7 + \
            [ctypes.c_uint32] + [ctypes.c_void_p] * 3 + [ctypes.c_uint32, ctypes.c_uint32]
        lib.oracle_mem_candidates.restype = ctypes.c_int
        lib.oracle_mem_candidates.argtypes = [ctypes.c_uint32] + [ctypes.c_void_p] * 3 + [ctypes.c_uint32] * 2 + \
            [ctypes.c_void_p]
        lib.oracle_memopt.restype = ctypes.c_int
        lib.oracle_memopt.argtypes = [ctypes.POINTER(_OProblem), ctypes.c_uint32] + [ctypes.c_void_p] * 3 + \
            [ctypes.c_uint32, ctypes.POINTER(_OCands), ctypes.c_uint64, ctypes.c_uint64] + [ctypes.c_void_p] * 7 + \
            [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p]
        lib.oracle_mcts_table.restype = ctypes.c_uint32
        lib.oracle_mcts_table.argtypes = [ctypes.c_uint32, ctypes.c_uint64] + [ctypes.c_uint32] * 3 + \
            [ctypes.c_double] * 2 + [ctypes.c_void_p] * 7 + [ctypes.c_uint32]
        lib.oracle_select_rank.restype = ctypes.c_int
        lib.oracle_select_rank.argtypes = [ctypes.c_uint32] + [ctypes.c_void_p] * 4 + \
            [ctypes.c_uint32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_argmin.restype = ctypes.c_int64
        lib.oracle_argmin.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64]
        _lib = lib
    return _lib


def chunk_layers(L: int, P: int, K: int):
    """O1 (R-3): layers per chunk, or None if P*K > L (TooManyChunks)."""
    out = np.zeros(max(1, P * K), np.uint32)
    rc = _load().oracle_chunk_layers(L, P, K, out.ctypes.data)
    return None if rc != 0 else [int(v) for v in out[:P * K]]


def split_sizes(N: int, M: int):
    """O2 (R-2): sizes of the M balanced contiguous parts of N instances."""
    st = np.zeros(M + 1, np.uint32)
    _load().oracle_split(N, M, st.ctypes.data)
    return [int(st[j + 1] - st[j]) for j in range(M)]


class _Bound:
    """Keeps the numpy arrays alive while C holds pointers into them."""

    def __init__(self, pb, cands, orders=None):
        from gen.problem import problem_arrays
        a = problem_arrays(pb)
        self.keep = dict(a)
        self.keep["inst_off"] = np.ascontiguousarray(pb.inst_off, np.uint32)
        self.keep["inst_units"] = np.ascontiguousarray(pb.inst_units, np.uint16)
        self.keep["budget_kib"] = np.ascontiguousarray(pb.budget_kib, np.uint32)
        k = self.keep
        self.pb = _OProblem(pb.P, pb.nmod, pb.m, *[k[n].ctypes.data for n in (
            "L", "K", "max_split", "w_max", "producer_mask", "tab_off", "tab_f", "tab_b", "tab_act", "tab_p2p",
            "chunk_off", "chunk_layers", "inst_off", "inst_units", "budget_kib")])
        self.c = cands
        self.ord = None if orders is None else np.ascontiguousarray(orders, np.uint16)
        if self.ord is not None:
            assert self.ord.shape == (cands.count, pb.P, 2 * pb.n_max), self.ord.shape
        self.cs = _OCands(pb.n_max, pb.fbw, *[np.ascontiguousarray(getattr(cands, n)).ctypes.data
                                              for n in ("split", "n", "fwd", "bwd", "fb")],
                          None if self.ord is None else self.ord.ctypes.data)


class Results:
    def __init__(self, count: int, P: int):
        self.makespan = np.zeros(count, np.uint64)
        self.status = np.zeros(count, np.uint32)
        self.oom_mask = np.zeros(count, np.uint32)
        self.bubble = np.zeros(count, np.float64)
        self.peaks = np.zeros((count, P), np.uint64)
        self.busy = np.zeros(count, np.uint64)


def evaluate(pb, cands, first: int = 0, count: Optional[int] = None, threads: int = 1, orders=None) -> Results:
    """O1-O10 for candidates [first, first+count) of the host-view batch `cands`; with `orders`
    ([count_total, P, 2 n_max] u16, segment id | 0x8000 for backward, 0xFFFF beyond 2n: explicit
    per-rank orders, f1's output) those replace the shared sequences + F/B bits (O4/O5)."""
    for n in ("split", "n", "fwd", "bwd", "fb"):
        assert getattr(cands, n).flags["C_CONTIGUOUS"], n
    if count is None:
        count = cands.count - first
    lib = _load()
    bd = _Bound(pb, cands, orders)
    res = Results(count, pb.P)
    lib.oracle_eval(ctypes.byref(bd.pb), ctypes.byref(bd.cs), first, count, res.makespan.ctypes.data,
                    res.status.ctypes.data, res.oom_mask.ctypes.data, res.bubble.ctypes.data,
                    res.peaks.ctypes.data, res.busy.ctypes.data, threads)
    return res


def interleave(pb, cands, first: int = 0, count: Optional[int] = None, threads: int = 1):
    """I1-I6: DIP's dual-queue greedy interleaving of each candidate's split and
    forward / backward priority orders (its F/B bits are ignored). Returns (orders, Results):
    orders [count, P, 2 n_max] u16 -- each rank's stage order, segment id | 0x8000 for a backward
    stage, 0xFFFF beyond 2n -- and the score of the built schedule."""
    for nme in ("split", "n", "fwd", "bwd", "fb"):
        assert getattr(cands, nme).flags["C_CONTIGUOUS"], nme
    if count is None:
        count = cands.count - first
    lib = _load()
    bd = _Bound(pb, cands)
    res = Results(count, pb.P)
    ords = np.zeros((count, pb.P, 2 * pb.n_max), np.uint16)
    rc = lib.oracle_interleave(ctypes.byref(bd.pb), ctypes.byref(bd.cs), first, count, ords.ctypes.data,
                               res.makespan.ctypes.data, res.status.ctypes.data, res.oom_mask.ctypes.data,
                               res.bubble.ctypes.data, res.peaks.ctypes.data, res.busy.ctypes.data, threads)
    assert rc == 0
    return ords, res


def mcts_table(Cn: int, seed: int, rounds: int, leaves: int, rollouts: int, alpha: float, beta: float, table,
               policy: int = 0):
    """S4-S6 alone with rollouts scored by table[seq[0], seq[1]] (a test fixture):
    returns dict(trace [rounds], leaves [rounds, leaves] node ids, tree: parent, cls, N, s per node).
    policy: 0 MCTS, 1 random exploration, 2 depth-first (P:963-972's comparison)."""
    t = np.ascontiguousarray(np.asarray(table, np.float64).reshape(-1))
    assert t.size == Cn * Cn
    cap = 1 + rounds * leaves
    trace = np.zeros(rounds, np.float64)
    lv = np.zeros((rounds, leaves), np.int32)
    par, cls, N, sv = np.zeros(cap, np.int32), np.zeros(cap, np.int32), np.zeros(cap, np.uint32), np.zeros(cap, np.float64)
    lib = _load()
    nn = lib.oracle_mcts_table(Cn, seed & ((1 << 64) - 1), rounds, leaves, rollouts, alpha, beta, t.ctypes.data,
                               trace.ctypes.data, lv.ctypes.data, par.ctypes.data, cls.ctypes.data, N.ctypes.data,
                               sv.ctypes.data, policy)
    return dict(trace=trace, leaves=lv, parent=par[:nn], cls=cls[:nn], N=N[:nn], s=sv[:nn])


def search(pb, split, seed: int, rounds: int, leaves: int, rollouts: int, alpha: float = 1.0, beta: float = 0.5,
           menu=None, S: int = 10, policy: int = 0):
    """S1-S6: MCTS over class orders with batched rounds, scoring rollouts with I1-I6
    (then M1-M4 if a strategy menu (f, b, act) is given); policy 1 / 2 = the random / depth-first
    exploration the paper compares against. Returns dict(score, makespan, trace, fwd,
    bwd, orders, scored)."""
    from gen import Candidates
    lib = _load()
    dummy = Candidates(pb, 1)
    bd = _Bound(pb, dummy)
    sp = np.ascontiguousarray(np.asarray(split, np.uint8).reshape(-1))
    trace = np.zeros(rounds, np.float64)
    sc = ctypes.c_double()
    mk = ctypes.c_uint64()
    scored = ctypes.c_uint64()
    fwd = np.zeros(pb.n_max, np.uint16)
    bwd = np.zeros(pb.n_max, np.uint16)
    ords = np.zeros((pb.P, 2 * pb.n_max), np.uint16)
    arrs = _menu_arrays(menu)                     # kept alive for the call
    lib.oracle_search(ctypes.byref(bd.pb), pb.n_max, pb.fbw, sp.ctypes.data, seed & ((1 << 64) - 1), rounds, leaves,
                      rollouts, alpha, beta, trace.ctypes.data, ctypes.byref(sc), ctypes.byref(mk), fwd.ctypes.data,
                      bwd.ctypes.data, ords.ctypes.data, ctypes.byref(scored), *_menu_args(arrs, S), policy)
    return dict(score=sc.value, makespan=mk.value, trace=trace, fwd=fwd, bwd=bwd, orders=ords, scored=scored.value)


def timeline(pb, cands, x: int, orders=None):
    """Per-(rank, slot) (start, end) arrays of candidate x, shape [P, 2n]; None unless timed
    (`orders`: explicit per-rank orders, as evaluate)."""
    lib = _load()
    bd = _Bound(pb, cands, orders)
    n = int(cands.n[x])
    st = np.zeros(max(1, pb.P * 2 * n), np.uint64)
    en = np.zeros_like(st)
    status = lib.oracle_timeline(ctypes.byref(bd.pb), ctypes.byref(bd.cs), x, st.ctypes.data, en.ctypes.data)
    if status not in (ST_OK, ST_OOM):
        return status, None, None
    return status, st[:pb.P * 2 * n].reshape(pb.P, 2 * n), en[:pb.P * 2 * n].reshape(pb.P, 2 * n)


def _menu_arrays(menu):
    """contiguous uint32 (f, b, act) of a strategy menu, or None"""
    return None if menu is None else tuple(np.ascontiguousarray(v, np.uint32) for v in menu)


def _menu_args(arrs, S):
    if arrs is None:
        return (0, None, None, None, S)
    f, b, a = arrs
    return (f.shape[0], f.ctypes.data, b.ctypes.data, a.ctypes.data, S)


def mem_candidates(f, b, act, layers: int, S: int):
    """M2: the <= S (F ns, B ns, mem KiB) candidates of a stage pair of `layers`
    identical layers whose per-layer strategy menu is (f[c], b[c], act[c]); sorted by memory."""
    f = np.ascontiguousarray(f, np.uint32)
    b = np.ascontiguousarray(b, np.uint32)
    a = np.ascontiguousarray(act, np.uint32)
    out = np.zeros((max(S, 2), 3), np.uint64)
    k = _load().oracle_mem_candidates(len(f), f.ctypes.data, b.ctypes.data, a.ctypes.data, layers, S,
                                      out.ctypes.data)
    return [tuple(int(v) for v in out[x]) for x in range(k)]


def select_rank(sF, sB, cands, budget: int, gap_pm: int = 50, node_cap: int = 4096):
    """M3 on one rank: pairs in forward order with slots sF[p] < ... and backward slots
    sB[p]; cands[p] = [(F, B, mem), ...] sorted by memory ascending. Returns (selection, stats)
    with stats = dict(warm, bound, final, nodes, infeasible, certified, capped)."""
    n = len(sF)
    Sst = max([len(c) for c in cands] + [1])
    arr = np.zeros((max(n, 1), Sst, 3), np.uint64)
    nc = np.zeros(max(n, 1), np.uint32)
    for p, cl in enumerate(cands):
        nc[p] = len(cl)
        for c, v in enumerate(cl):
            arr[p, c] = v
    f = np.ascontiguousarray(sF, np.uint32)
    b = np.ascontiguousarray(sB, np.uint32)
    cur = np.zeros(max(n, 1), np.uint32)
    st = np.zeros(5, np.uint64)
    _load().oracle_select_rank(n, f.ctypes.data, b.ctypes.data, nc.ctypes.data, arr.ctypes.data, Sst, int(budget),
                               gap_pm, node_cap, cur.ctypes.data, st.ctypes.data)
    fl = int(st[4])
    return [int(v) for v in cur[:n]], {"warm": int(st[0]), "bound": int(st[1]), "final": int(st[2]),
                                       "nodes": int(st[3]), "infeasible": bool(fl & 1),
                                       "certified": bool(fl & 2), "capped": bool(fl & 4)}


def memopt(pb, cands, menu, S: int = 10, first: int = 0, count: Optional[int] = None, threads: int = 1,
           gap_pm: int = 50, node_cap: int = 4096, stats: bool = False, orders=None):
    """M1-M4: per-layer memory optimisation of each candidate schedule. `menu` =
    (f, b, act) arrays [n_strat, T] aligned with the model's tables. Returns (sel, Results) with
    sel [count, P, 2, n_max] the selected candidate index of each pair at forward position p
    (sel[..., 0, p]) and backward position q (sel[..., 1, q]) and the re-timed results. M3 solves
    each rank's ILP to a relative gap <= gap_pm per mille, at most node_cap B&B children.
    With stats=True also returns [count, P, 5] per-rank (warm, bound, final, nodes, flags). With
    `orders` (explicit per-rank orders, as evaluate) the pairs come from those orders."""
    if count is None:
        count = cands.count - first
    f, b, a = (np.ascontiguousarray(v, np.uint32) for v in menu)
    lib = _load()
    bd = _Bound(pb, cands, orders)
    res = Results(count, pb.P)
    sel = np.zeros((count, pb.P, 2, pb.n_max), np.uint8)
    rst = np.zeros((count, pb.P, 5), np.uint64) if stats else None
    rc = lib.oracle_memopt(ctypes.byref(bd.pb), f.shape[0], f.ctypes.data, b.ctypes.data, a.ctypes.data, S,
                           ctypes.byref(bd.cs), first, count, sel.ctypes.data, res.makespan.ctypes.data,
                           res.status.ctypes.data, res.oom_mask.ctypes.data, res.bubble.ctypes.data,
                           res.peaks.ctypes.data, res.busy.ctypes.data, threads, gap_pm, node_cap,
                           None if rst is None else rst.ctypes.data)
    assert rc == 0
    return (sel, res, rst) if stats else (sel, res)


def argmin(makespan: np.ndarray, status: np.ndarray) -> int:
    """O11 (R-14, R-15): lowest index among the OK candidates of minimal makespan."""
    ms = np.ascontiguousarray(makespan, np.uint64)
    st = np.ascontiguousarray(status, np.uint32)
    return int(_load().oracle_argmin(ms.ctypes.data, st.ctypes.data, len(ms)))
