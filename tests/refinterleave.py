"""A second, independent dual-queue interleaver (§5.2) used only to cross-check
the oracle's I1-I6 on small cases.

Differs from oracle/dip_oracle.c on purpose: no indegree counting and no ready lists -- every step
re-derives, for every rank, which of its unscheduled stages are ready by asking a recursive
predecessor function whether all predecessors are scheduled, and recomputes their start times from
scratch. Same readings (R-29..R-31). Pure Python, for small P*2n only.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

from tests.refsim import _layers, _split_sizes


def interleave(pb, cs, x: int):
    """Returns (per-rank orders as lists of ('F'|'B', segment id), makespan, peaks, oom flag), or
    None for a malformed candidate."""
    P, m, nm = pb.P, pb.m, pb.nmod
    mods = pb.modules
    split = cs.split[x].reshape(m, nm).astype(int)
    Ninst = pb.n_inst()
    base = pb.seg_base()
    W: Dict[int, int] = {}
    dec: Dict[int, Tuple[int, int, int, int]] = {}
    for b in range(m):
        for i, md in enumerate(mods):
            N, M = int(Ninst[b, i]), int(split[b, i])
            if (N == 0) != (M == 0) or M > min(N, md.max_split):
                return None
            if M == 0:
                continue
            lo = int(pb.inst_off[b * nm + i])
            acc = 0
            for j, sz in enumerate(_split_sizes(N, M)):
                w = int(pb.inst_units[lo + acc:lo + acc + sz].astype(np.int64).sum())
                acc += sz
                for k in range(md.K):
                    s = int(base[b, i]) + j * md.K + k
                    W[s] = w
                    dec[s] = (b, i, j, k)
    n = len(W)
    if int(cs.n[x]) != n:
        return None
    fwd = [int(v) for v in cs.fwd[x, :n]]
    bwd = [int(v) for v in cs.bwd[x, :n]]
    if sorted(fwd) != sorted(W) or sorted(bwd) != sorted(W):
        return None
    prio = {(0, s): p for p, s in enumerate(fwd)}
    prio.update({(1, s): p for p, s in enumerate(bwd)})

    def cost(d, s, r):
        b, i, j, k = dec[s]
        md = mods[i]
        lay = _layers(pb, i, k * P + r)
        w = W[s]
        return lay * int(md.b_ns[w] if d else md.f_ns[w]), lay * int(md.act_kib[w]), int(md.p2p_ns[w])

    def preds(d, s, r):
        b, i, j, k = dec[s]
        md = mods[i]
        out = []
        if d == 0:
            if r > 0:
                out.append(((0, s, r - 1), cost(0, s, r)[2]))
            elif k > 0:
                out.append(((0, s - 1, P - 1), cost(0, s - 1, 0)[2] if P > 1 else 0))
            else:
                for p in range(nm):
                    if (md.producer_mask >> p) & 1:
                        for jp in range(int(split[b, p])):
                            pr = int(base[b, p]) + jp * mods[p].K + mods[p].K - 1
                            out.append(((0, pr, P - 1), cost(0, pr, 0)[2] if P > 1 else 0))
        else:
            if r + 1 < P:
                out.append(((1, s, r + 1), cost(0, s, 0)[2]))
            elif k + 1 < md.K:
                out.append(((1, s + 1, 0), cost(0, s, 0)[2] if P > 1 else 0))
            else:
                cons = [(c, jc) for c in range(nm) if (mods[c].producer_mask >> i) & 1 for jc in range(int(split[b, c]))]
                for c, jc in cons:
                    out.append(((1, int(base[b, c]) + jc * mods[c].K, 0), cost(0, s, 0)[2] if P > 1 else 0))
                if not cons:
                    out.append(((0, s, P - 1), 0))
        return out

    end: Dict[Tuple[int, int, int], int] = {}
    todo = [{(d, s) for d in (0, 1) for s in W} for _ in range(P)]
    tlast, last, cur, peak = [0] * P, [-1] * P, [0] * P, [0] * P
    order: List[List[Tuple[str, int]]] = [[] for _ in range(P)]
    bud = [int(v) for v in pb.budget_kib]

    def tstart(d, s, r):
        t = 0
        for node, w in preds(d, s, r):
            if node not in end:
                return None
            t = max(t, end[node] + w)
        return t

    while any(todo):
        ready = []
        for r in range(P):
            rd = {}
            for d, s in todo[r]:
                t = tstart(d, s, r)
                if t is not None:
                    rd[(d, s)] = t
            ready.append(rd)
        choice = None
        for relax in (False, True):
            best = None
            for r in range(P):
                ts = [t for (d, s), t in ready[r].items()
                      if d == 1 or relax or cur[r] + cost(0, s, r)[1] <= bud[r]]
                if relax:
                    ts = [t for (d, s), t in ready[r].items() if d == 0]
                if ts and (best is None or min(ts) < best[0]):
                    best = (min(ts), r)
            if best is not None:
                choice = (best[1], relax)
                break
        if choice is None:
            return None
        r, relax = choice
        F = {s: t for (d, s), t in ready[r].items() if d == 0 and (relax or cur[r] + cost(0, s, r)[1] <= bud[r])}
        B = {s: t for (d, s), t in ready[r].items() if d == 1}
        tf = min(F.values()) if F else None
        tb = min(B.values()) if B else None
        if tf is not None and tb is not None and tf < tlast[r] and tb < tlast[r]:
            d = 1 if last[r] == 0 else 0
        elif tf is None:
            d = 1
        elif tb is None:
            d = 0
        else:
            d = 1 if tb <= tf else 0
        pool = B if d else F
        lim = max(tb if d else tf, tlast[r])
        s = min((prio[(d, s)], s) for s, t in pool.items() if t <= lim)[1]
        t0 = pool[s]
        lat, act, _ = cost(d, s, r)
        st = max(t0, tlast[r])
        end[(d, s, r)] = st + lat
        tlast[r] = st + lat
        last[r] = d
        todo[r].discard((d, s))
        order[r].append(("B" if d else "F", s))
        if d:
            cur[r] -= act
        else:
            cur[r] += act
            peak[r] = max(peak[r], cur[r])
    mk = max(end.values()) if end else 0
    return order, mk, peak, any(peak[r] > bud[r] for r in range(P))
