"""Lock-step round counts of the record scorer on generated candidates (CPU simulation): lane = rank
(the kernel) vs two ranks per lane processed in alternating order within a round, and vs a lane
retiring up to R consecutive ready stages per round (rounds, and inner iterations = the sum over
rounds of the most stages any lane retired: what a warp would execute). Used for DESIGN.md §6 / §9.
  PYTHONPATH=. python scripts/lockstep_rounds.py 94B 6"""
import numpy as np, gen, sys
sys.path.insert(0, '/root/repo')
from tests.refsim import _split_sizes

def orders_and_deps(pb, cs, x):
    P, m, nm = pb.P, pb.m, pb.nmod
    split = cs.split[x].reshape(m, nm).astype(int); base = pb.seg_base(); mods = pb.modules
    n = int(cs.n[x]); fwd = [int(v) for v in cs.fwd[x, :n]]; bwd = [int(v) for v in cs.bwd[x, :n]]
    dec = {}
    for b in range(m):
        for i, md in enumerate(mods):
            for j in range(split[b, i]):
                for k in range(md.K): dec[int(base[b, i]) + j * md.K + k] = (b, i, j, k)
    ords = []
    for r in range(P):
        fi = bi = 0; row = []
        for t in range(2 * n):
            if (int(cs.fb[x, r, t >> 5]) >> (t & 31)) & 1: row.append((1, bwd[bi])); bi += 1
            else: row.append((0, fwd[fi])); fi += 1
        ords.append(row)
    def preds(d, s, r):
        b, i, j, k = dec[s]; md = mods[i]; out = []
        if d == 0:
            if r > 0: out.append((0, s, r - 1))
            elif k > 0: out.append((0, s - 1, P - 1))
            else:
                for p in range(nm):
                    if (md.producer_mask >> p) & 1:
                        for jp in range(split[b, p]): out.append((0, int(base[b, p]) + jp * mods[p].K + mods[p].K - 1, P - 1))
        else:
            if r + 1 < P: out.append((1, s, r + 1))
            elif k + 1 < md.K: out.append((1, s + 1, 0))
            else:
                cons = [(c, jc) for c in range(nm) if (mods[c].producer_mask >> i) & 1 for jc in range(split[b, c])]
                for c, jc in cons: out.append((1, int(base[b, c]) + jc * mods[c].K, 0))
                if not cons: out.append((0, s, P - 1))
        return out
    return ords, preds, n

def rounds_lockstep(P, ords, preds, n, pair=False):
    done = {}; cur = [0] * P; rnd = 0
    total = sum(len(o) for o in ords)
    placed = 0
    while placed < total:
        rnd += 1
        if not pair:
            snap = dict(done)
            for r in range(P):
                if cur[r] < len(ords[r]):
                    d, s = ords[r][cur[r]]
                    if all(p in snap for p in preds(d, s, r)):
                        done[(d, s, r)] = rnd; cur[r] += 1; placed += 1
        else:
            snap = dict(done)
            for l in range(0, P, 2):
                seq = [l, l + 1] if rnd % 2 else [l + 1, l]
                local = dict(snap)   # lane-local visibility: its own ranks' results this round
                for r in seq:
                    if r >= P or cur[r] >= len(ords[r]): continue
                    d, s = ords[r][cur[r]]
                    if all(p in local for p in preds(d, s, r)):
                        done[(d, s, r)] = rnd; local[(d, s, r)] = rnd; cur[r] += 1; placed += 1
        if rnd > 100000: return None
    return rnd

def rounds_multi(P, ords, preds, R):
    done = set(); cur = [0] * P; rnd = 0; iters = 0
    total = sum(len(o) for o in ords); placed = 0
    while placed < total:
        rnd += 1; snap = set(done); mx = 0
        for r in range(P):
            k = 0
            while k < R and cur[r] < len(ords[r]):
                d, s = ords[r][cur[r]]
                if not all((p in snap) or (p[2] == r and p in done) for p in preds(d, s, r)): break
                done.add((d, s, r)); cur[r] += 1; placed += 1; k += 1
            mx = max(mx, k)
        iters += max(mx, 1)
        if rnd > 100000: return None
    return rnd, iters

pb = gen.make_problem(sys.argv[1]); N = int(sys.argv[2])
cs = gen.generate(pb, 0, N, p_mutate=0, p_bad=0)
a = []; b = []
for x in range(N):
    ords, preds, n = orders_and_deps(pb, cs, x)
    r1 = rounds_lockstep(pb.P, ords, preds, n)
    r2 = rounds_lockstep(pb.P, ords, preds, n, pair=True)
    if r1 and r2: a.append(r1); b.append(r2); print(x, 2 * n, r1, r2, "multi (R: rounds, iterations)",
                                                   {R: rounds_multi(pb.P, ords, preds, R) for R in (2, 4, 1000)})
print("mean slots", np.mean([2 * int(cs.n[x]) for x in range(N)]), "lockstep", np.mean(a), "pair", np.mean(b))
