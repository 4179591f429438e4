"""Test-only builders: hand problems and textbook schedules (1F1B, GPipe, VPP).

These construct INPUTS (problems and host-view candidates) for the pins of
SURVEY.md Appendix A; they compute no timing.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from gen import Candidates, Module, Problem


def table(w_max: int, entries: Dict[int, Tuple[int, int, int, int]]):
    """Per-layer table arrays (F, B, act, p2p) with the given W -> values, zeros elsewhere."""
    f = np.zeros(w_max + 1, np.uint32)
    b = np.zeros_like(f)
    a = np.zeros_like(f)
    p = np.zeros_like(f)
    for w, (fv, bv, av, pv) in entries.items():
        f[w], b[w], a[w], p[w] = fv, bv, av, pv
    return f, b, a, p


def uniform_problem(P: int, m: int, tf: int, tb: int, act: int = 1, p2p: int = 0, K: int = 1,
                    layers_per_chunk: int = 1, budget: Optional[Sequence[int]] = None) -> Problem:
    """One module, K segments, every microbatch one instance of 1 unit: per-stage F=tf, B=tb."""
    L = P * K * layers_per_chunk
    md = Module("m", L, K, 1, 1, 0, *table(1, {1: (tf, tb, act, p2p)}))
    off = np.arange(m + 1, dtype=np.uint32)
    units = np.ones(m, np.uint16)
    bud = np.array(budget if budget is not None else [1 << 31] * P, np.uint32)
    return Problem("uniform", P, m, [md], off, units, bud)


def candidates_from_orders(pb: Problem, splits: Sequence[Sequence[int]],
                           orders: List[List[List[Tuple[str, int]]]]) -> Candidates:
    """orders[c][r] = list of ('F'|'B', segment id) for rank r of candidate c.

    fwd_seq / bwd_seq are read off rank 0 (all ranks must share them, reading R-1)."""
    cs = Candidates(pb, len(orders))
    for c, (sp, rk) in enumerate(zip(splits, orders)):
        cs.split[c] = np.asarray(sp, np.uint8).reshape(-1)
        fseq = [s for d, s in rk[0] if d == "F"]
        bseq = [s for d, s in rk[0] if d == "B"]
        n = len(fseq)
        cs.n[c] = n
        cs.fwd[c, :n] = fseq
        cs.bwd[c, :n] = bseq
        for r in range(pb.P):
            assert [s for d, s in rk[r] if d == "F"] == fseq, "ranks must share fwd_seq"
            assert [s for d, s in rk[r] if d == "B"] == bseq, "ranks must share bwd_seq"
            for t, (d, _) in enumerate(rk[r]):
                if d == "B":
                    cs.fb[c, r, t >> 5] |= np.uint32(1 << (t & 31))
    return cs


def one_f_one_b(P: int, m: int) -> List[List[Tuple[str, int]]]:
    """Megatron 1F1B: rank r warms up with min(P-r, m) forwards, then alternates B/F (R-17)."""
    out = []
    for r in range(P):
        w = min(P - r, m)
        seq = [("F", i) for i in range(w)]
        f, b = w, 0
        while b < m:
            seq.append(("B", b))
            b += 1
            if f < m:
                seq.append(("F", f))
                f += 1
        out.append(seq)
    return out


def gpipe(P: int, m: int) -> List[List[Tuple[str, int]]]:
    return [[("F", i) for i in range(m)] + [("B", i) for i in range(m)] for _ in range(P)]


def vpp(P: int, v: int, m: int) -> List[List[Tuple[str, int]]]:
    """Megatron interleaved 1F1B for one module with K = v segments.

    Segment id of (microbatch b, chunk k) is b*v + k (id scheme with M_max = 1).
    Forward virtual microbatch x -> chunk (x mod P*v) div P, microbatch (x div P*v)*P + x mod P;
    backward uses chunk v-1-((x mod P*v) div P).  Rank r: min((P-r-1)*2 + (v-1)*P, m*v) warm-up
    forwards, then alternate F, B."""
    tot = m * v

    def fseg(x):
        ch = (x % (P * v)) // P
        mb = (x // (P * v)) * P + x % P
        return mb * v + ch

    def bseg(x):
        ch = v - 1 - (x % (P * v)) // P
        mb = (x // (P * v)) * P + x % P
        return mb * v + ch

    out = []
    for r in range(P):
        w = min((P - r - 1) * 2 + (v - 1) * P, tot)
        if v == 1:
            w = min(P - r, m)
        seq = [("F", fseg(x)) for x in range(w)]
        f, b = w, 0
        while b < tot:
            if f < tot and v > 1:
                seq.append(("F", fseg(f)))
                f += 1
            seq.append(("B", bseg(b)))
            b += 1
            if v == 1 and f < tot:
                seq.append(("F", fseg(f)))
                f += 1
        out.append(seq)
    return out


def diamond_problem(P: int = 4, m: int = 6, seed: int = 0) -> Problem:
    """Four modules in a diamond: vision (M_max 4) and audio (M_max 2) both feed a fusion module
    (K = 2, M_max 2) that feeds an LLM (K = 2) -- joins with several producer modules and split
    sub-microbatches on both sides, some microbatches without vision or audio instances."""
    rng = np.random.default_rng(seed)
    w = 8

    def tab(scale):
        return table(w, {u: (scale * u + 5, 2 * scale * u + 9, 3 * u, u) for u in range(1, w + 1)})

    mods = [Module("vision", 2 * P, 1, 4, w, 0, *tab(7)),
            Module("audio", P, 1, 2, w, 0, *tab(5)),
            Module("fusion", 2 * P * 2, 2, 2, w, 0b011, *tab(3)),
            Module("llm", 4 * P, 2, 1, w, 0b100, *tab(11))]
    units, off = [], [0]
    for b in range(m):
        nv = int(rng.integers(0, 5)) if b % 3 else 0          # every third microbatch: no vision
        na = int(rng.integers(0, 3))
        per = [[int(rng.integers(1, 3)) for _ in range(nv)], [int(rng.integers(1, 5)) for _ in range(na)],
               [int(rng.integers(1, 5)) for _ in range(int(rng.integers(1, 3)))], [int(rng.integers(1, 9))]]
        for lst in per:
            units += lst
            off.append(len(units))
    return Problem("diamond", P, m, mods, np.array(off, np.uint32), np.array(units, np.uint16),
                   np.full(P, 700, np.uint32))


def orders_array(pb: Problem, rank_orders: List[List[Tuple[str, int]]]) -> np.ndarray:
    """[P, 2 n_max] u16 per-rank orders (segment id | 0x8000 for backward, 0xFFFF padding) from
    lists of ('F'|'B', segment id) -- the f1 output format."""
    out = np.full((pb.P, 2 * pb.n_max), 0xFFFF, np.uint16)
    for r, seq in enumerate(rank_orders):
        for t, (d, s) in enumerate(seq):
            out[r, t] = s | (0x8000 if d == "B" else 0)
    return out


def orders_lists(ords: np.ndarray) -> List[List[Tuple[str, int]]]:
    """inverse of orders_array for one candidate"""
    return [[("B" if v & 0x8000 else "F", int(v) & 0x7FFF) for v in row if v != 0xFFFF] for row in ords]
