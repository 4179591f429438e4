"""A second, independent evaluator used only to cross-check the oracle on small cases.

Differs from oracle/dip_oracle.c on purpose: no explicit edge list and no Kahn
queue. Each node's end time is a memoised recursive longest-path over an
implicit dependency function; a node met again while on the recursion stack is
a cycle (DEADLOCK). Pure Python, for small P*2n only.
"""
from __future__ import annotations

import sys
from typing import Dict, List, Optional, Tuple

import numpy as np

OK, OOM, DEADLOCK, BAD = 0, 1, 2, 3


def _split_sizes(N: int, M: int) -> List[int]:
    # balanced contiguous parts, the first N mod M get one more (reading R-2)
    return [N // M + (1 if j < N % M else 0) for j in range(M)]


def _layers(pb, i: int, c: int) -> int:
    md = pb.modules[i]
    if md.chunk_layers is not None:
        return int(md.chunk_layers[c])
    C = pb.P * md.K
    return md.L // C + (1 if c < md.L % C else 0)


def evaluate(pb, cs, x: int):
    """Returns (status, makespan or None, peaks list, bubble, busy)."""
    P, m, nm = pb.P, pb.m, pb.nmod
    mods = pb.modules
    split = cs.split[x].reshape(m, nm).astype(int)
    Ninst = pb.n_inst()
    base = pb.seg_base()
    # parts and work units
    W: Dict[int, int] = {}
    dec: Dict[int, Tuple[int, int, int, int]] = {}
    for b in range(m):
        for i, md in enumerate(mods):
            N, M = int(Ninst[b, i]), int(split[b, i])
            if (N == 0) != (M == 0) or M > min(N, md.max_split):
                return BAD, None, [0] * P, -1.0, 0
            if M == 0:
                continue
            lo = int(pb.inst_off[b * nm + i])
            pos = lo
            for j, sz in enumerate(_split_sizes(N, M)):
                w = int(sum(int(u) for u in pb.inst_units[pos:pos + sz]))
                pos += sz
                for k in range(md.K):
                    sid = int(base[b, i]) + j * md.K + k
                    W[sid] = w
                    dec[sid] = (b, i, j, k)
    n = len(W)
    if int(cs.n[x]) != n:
        return BAD, None, [0] * P, -1.0, 0
    fseq = [int(v) for v in cs.fwd[x][:n]]
    bseq = [int(v) for v in cs.bwd[x][:n]]
    if sorted(fseq) != sorted(W) or sorted(bseq) != sorted(W):
        return BAD, None, [0] * P, -1.0, 0
    if any(int(v) != 0xFFFF for v in cs.fwd[x][n:]) or any(int(v) != 0xFFFF for v in cs.bwd[x][n:]):
        return BAD, None, [0] * P, -1.0, 0
    orders = []
    for r in range(P):
        bits = [(int(cs.fb[x, r, t >> 5]) >> (t & 31)) & 1 for t in range(32 * pb.fbw)]
        if sum(bits[:2 * n]) != n or any(bits[2 * n:]):
            return BAD, None, [0] * P, -1.0, 0
        fi = bi = 0
        o = []
        for t in range(2 * n):
            if bits[t]:
                o.append(("B", bseq[bi]))
                bi += 1
            else:
                o.append(("F", fseq[fi]))
                fi += 1
        orders.append(o)
    if n == 0:
        return OK, 0, [0] * P, 0.0, 0
    slot = {}
    for r in range(P):
        for t, (d, s) in enumerate(orders[r]):
            slot[(d, s, r)] = t

    def cost(d, s, r):
        b, i, j, k = dec[s]
        T = mods[i]
        lay = _layers(pb, i, k * P + r)
        lat = lay * int(T.f_ns[W[s]] if d == "F" else T.b_ns[W[s]])
        return lat, lay * int(T.act_kib[W[s]]), int(T.p2p_ns[W[s]])

    def deps(d, s, r):
        """(dir, seg, rank, weight) predecessors other than the previous slot."""
        b, i, j, k = dec[s]
        K = mods[i].K
        wr = lambda seg: cost("F", seg, 0)[2] if P > 1 else 0  # noqa: E731
        out = []
        if d == "F":
            if r > 0:
                out.append(("F", s, r - 1, cost("F", s, r)[2]))
            elif k > 0:
                out.append(("F", s - 1, P - 1, wr(s - 1)))
            else:
                for ip in range(nm):
                    if (mods[i].producer_mask >> ip) & 1:
                        for jp in range(int(split[b, ip])):
                            pr = int(base[b, ip]) + jp * mods[ip].K + mods[ip].K - 1
                            out.append(("F", pr, P - 1, wr(pr)))
        else:
            if r < P - 1:
                out.append(("B", s, r + 1, cost("F", s, r)[2]))
            elif k < K - 1:
                out.append(("B", s + 1, 0, wr(s)))
            else:
                cons = [(ic, jc) for ic in range(nm) if (mods[ic].producer_mask >> i) & 1
                        for jc in range(int(split[b, ic]))]
                for ic, jc in cons:
                    out.append(("B", int(base[b, ic]) + jc * mods[ic].K, 0, wr(s)))
                if not cons:
                    out.append(("F", s, P - 1, 0))
        return out

    end: Dict[Tuple[str, int, int], int] = {}
    onstack = set()
    sys.setrecursionlimit(max(10000, 8 * P * n + 100))

    class Cycle(Exception):
        pass

    def get_end(d, s, r):
        key = (d, s, r)
        if key in end:
            return end[key]
        if key in onstack:
            raise Cycle()
        onstack.add(key)
        t = slot[key]
        st = get_end(*orders[r][t - 1], r) if t > 0 else 0
        for dd, ss, rr, w in deps(d, s, r):
            st = max(st, get_end(dd, ss, rr) + w)
        onstack.discard(key)
        end[key] = st + cost(d, s, r)[0]
        return end[key]

    peaks = []
    oom = False
    for r in range(P):
        cur = pk = 0
        for d, s in orders[r]:
            a = cost(d, s, r)[1]
            if d == "F":
                cur += a
                pk = max(pk, cur)
            else:
                cur -= a
        peaks.append(pk)
        oom |= pk > int(pb.budget_kib[r])
    try:
        mk = max(get_end(d, s, r) for r in range(P) for d, s in orders[r])
    except Cycle:
        return DEADLOCK, None, peaks, -1.0, 0
    busy = sum(cost(d, s, r)[0] for r in range(P) for d, s in orders[r])
    den = P * mk
    bub = (den - busy) / den if den else 0.0
    return (OOM if oom else OK), mk, peaks, bub, busy
