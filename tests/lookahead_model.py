"""A model of the f1 kernel's step rule (csrc/dip_order.cu, BUILD), used only by tests: DIP's
dual-queue greedy (reading R-29) run serially -- one placement per step on the rank with
the smallest (t_min, rank) -- and with the kernel's conservative parallel steps, where every rank
whose key is below both ring neighbours' lower bounds places too (bounds relaxed `nit` times from
the step's smallest key, times relative to it and saturated at 2^31 - 1, as in the kernel). Both
must give the same per-rank orders; `run` also counts the steps.

    python -m tests.lookahead_model 94B 1
"""
from __future__ import annotations

import sys

import numpy as np

import gen
from tests.refsim import _layers, _split_sizes

INF = 1 << 62
CAP = (1 << 31) - 1


def build(pb, cs, x):
    P, m, nm = pb.P, pb.m, pb.nmod
    mods = pb.modules
    split = cs.split[x].reshape(m, nm).astype(int)
    Ninst = pb.n_inst()
    base = pb.seg_base()
    W, dec = {}, {}
    for b in range(m):
        for i, md in enumerate(mods):
            N, M = int(Ninst[b, i]), int(split[b, i])
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
    fwd = [int(v) for v in cs.fwd[x, :n]]
    bwd = [int(v) for v in cs.bwd[x, :n]]
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

    nodes = [(d, s, r) for r in range(P) for d in (0, 1) for s in W]
    pr = {v: preds(*v) for v in nodes}
    succ = {v: [] for v in nodes}
    for v, ps in pr.items():
        for u, w in ps:
            succ[u].append((v, w))
    # the kernel's per-rank lookahead: shortest stage of the rank + smallest p2p of any segment
    wmin = min(cost(0, s, 0)[2] for s in W) if W else 0
    dlt = [(min(min(cost(0, s, r)[0], cost(1, s, r)[0]) for s in W) + wmin) if W else 0 for r in range(P)]
    return dict(P=P, W=W, prio=prio, cost=cost, pr=pr, succ=succ, bud=[int(v) for v in pb.budget_kib],
                dlt=dlt)


class Sim:
    def __init__(self, g):
        self.g = g
        P = g["P"]
        self.wait = {v: len(ps) for v, ps in g["pr"].items()}
        self.rt = {v: 0 for v in g["pr"]}
        self.pool = [[{}, {}] for _ in range(P)]
        for v, c in self.wait.items():
            if c == 0:
                self.pool[v[2]][v[0]][v[1]] = 0
        self.tlast, self.last, self.cur = [0] * P, [-1] * P, [0] * P
        self.order = [[] for _ in range(P)]
        self.left = sum(1 for _ in g["pr"])
        self.todo = [2 * len(g["W"])] * P

    def keys(self, r, relax=False):
        cost, bud = self.g["cost"], self.g["bud"]
        F = {s: t for s, t in self.pool[r][0].items() if relax or self.cur[r] + cost(0, s, r)[1] <= bud[r]}
        B = self.pool[r][1]
        return F, B

    def key(self, r):
        F, B = self.keys(r)
        ts = list(F.values()) + list(B.values())
        return min(ts) if ts else None

    def place(self, r, relax):
        cost = self.g["cost"]
        F, B = self.keys(r, relax)
        tf = min(F.values()) if F else None
        tb = min(B.values()) if B else None
        tl = self.tlast[r]
        if tf is not None and tb is not None and tf < tl and tb < tl:
            d = 1 if self.last[r] == 0 else 0
        elif tf is None:
            d = 1
        elif tb is None:
            d = 0
        else:
            d = 1 if tb <= tf else 0
        pool = B if d else F
        lim = max(tb if d else tf, tl)
        s = min((self.g["prio"][(d, s)], s) for s, t in pool.items() if t <= lim)[1]
        t0 = pool[s]
        lat, act, _ = cost(d, s, r)
        st = max(t0, tl)
        end = st + lat
        self.tlast[r] = end
        self.last[r] = d
        del self.pool[r][d][s]
        self.order[r].append(("B" if d else "F", s))
        self.cur[r] += -act if d else act
        self.left -= 1
        self.todo[r] -= 1
        for v, w in self.g["succ"][(d, s, r)]:
            self.rt[v] = max(self.rt[v], end + w)
            self.wait[v] -= 1
            if self.wait[v] == 0:
                self.pool[v[2]][v[0]][v[1]] = self.rt[v]

    def pick_serial(self):
        P = self.g["P"]
        best = None
        for r in range(P):
            k = self.key(r)
            if k is not None and (best is None or k < best[0]):
                best = (k, r)
        if best is not None:
            return [best[1]], False
        best = None
        for r in range(P):
            ts = list(self.pool[r][0].values())
            if ts and (best is None or min(ts) < best[0]):
                best = (min(ts), r)
        return ([best[1]], True) if best else ([], False)

    def pick_parallel(self, nit=3):
        """the kernel's rule: (ranks placing in this step, relax)"""
        P = self.g["P"]
        ks = []
        for r in range(P):
            k = self.key(r)
            ks.append(INF if k is None else (k << 5) | r)
        if all(k == INF for k in ks) or P == 1:
            return self.pick_serial()
        gk = min(ks)
        g0 = gk >> 5
        kr = [CAP if k == INF else min((k >> 5) - g0, CAP) for k in ks]
        tr = [min(max(self.tlast[r] - g0, 0), CAP) for r in range(P)]
        dl = [min(v, CAP) for v in self.g["dlt"]]
        K = [0] * P
        for _ in range(nit):
            A = [CAP if self.todo[i] == 0 else min(max(tr[i], K[i]) + dl[i], CAP) for i in range(P)]
            K = [min(kr[j], A[(j - 1) % P], A[(j + 1) % P]) for j in range(P)]
        el = [r for r in range(P) if ks[r] != INF and
              (ks[r] == gk or (kr[r] < K[(r - 1) % P] and kr[r] < K[(r + 1) % P]))]
        return el, False

    def run(self, parallel, nit=3):
        steps = 0
        while self.left:
            rs, relax = self.pick_parallel(nit) if parallel else self.pick_serial()
            assert rs, "no rank can place"
            for r in rs:
                self.place(r, relax)
            steps += 1
        return steps


def compare(pb, cs, x, nit=3):
    """(serial steps, parallel steps); asserts identical per-rank orders"""
    g = build(pb, cs, x)
    a, b = Sim(g), Sim(g)
    ns, npar = a.run(False), b.run(True, nit)
    assert a.order == b.order, x
    return ns, npar


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "toy"
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    nit = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, mode=0, p_mutate=0.0, p_bad=0.0)
    ts = tp = 0
    for x in range(count):
        ns, npar = compare(pb, cs, x, nit)
        ts, tp = ts + ns, tp + npar
        print(f"x={x} serial steps {ns} parallel steps {npar} ({ns / npar:.2f}x)", flush=True)
    print(f"{name}: {ts / tp:.2f}x fewer steps")
