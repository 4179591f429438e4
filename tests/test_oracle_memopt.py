"""Pins of the oracle's per-layer memory optimisation (M1-M4, §5.3).

* M2 candidates: the worked examples of SPEC.md:416-417 ("2 layers x {none: (10 ms, 8 GB),
  checkpoint: (13 ms, 2 GB)}, S=3 -> {(20 ms, 16 GB), (23 ms, 10 GB), (26 ms, 4 GB)}"; "1 layer,
  2 strategies, S=10 -> exactly 2 candidates"), and properties against brute force over every
  per-layer assignment: extremes present, Pareto order, size <= S, and the bucket guarantee
  (every combination is matched by a candidate no slower and at most one bucket width larger);
* M3 selection (the per-rank ILP): SPEC.md:425-426's one-pair examples (M = 10 GB ->
  the 8 GB candidate, M = 12 GB -> the 6 ms one); unbounded memory -> every pair at its fastest
  candidate, whose re-timed makespan equals the fixed-order oracle run on the fastest strategy's
  tables; brute force over all selections of tiny ranks and tiny schedules: feasible, within the
  5 % gap of the optimum on EVERY instance, exactly optimal at gap 0, the bound never above
  the optimum; a hand-made instance where the greedy warm start is 36 % off and the branch and
  bound closes it; at full size against scipy's HiGHS ILP solver (within 5 % of its proven lower
  bound); on generated schedules an independent re-check of feasibility at every forward slot
  and, where the warm start is certified, of its termination (no single pair can still move up);
* M4: all pairs at candidate 0 reproduces the fixed-order oracle exactly.
"""
import itertools

import numpy as np
import pytest

import gen
import oracle
from gen import Candidates, Module, Problem
from gen.problem import problem_arrays, strategy_menu
from tests import helpers as H

GB = 1 << 20          # KiB


def test_candidates_spec_two_layer_example():
    # strategy 0 = checkpoint (13 ms, 2 GB), 1 = none (10 ms, 8 GB); F = 4 ms in both
    c = oracle.mem_candidates([4, 4], [9, 6], [2 * GB, 8 * GB], layers=2, S=3)
    assert [(f + b, m) for f, b, m in c] == [(26, 4 * GB), (23, 10 * GB), (20, 16 * GB)]


def test_candidates_spec_one_layer_extremes():
    c = oracle.mem_candidates([4, 2], [6, 4], [8 * GB, 12 * GB], layers=1, S=10)
    assert [(f + b, m) for f, b, m in c] == [(10, 8 * GB), (6, 12 * GB)]


def test_candidates_single_strategy():
    assert oracle.mem_candidates([5], [7], [3], layers=4, S=10) == [(20, 28, 12)]


@pytest.mark.parametrize("seed", range(40))
def test_candidates_properties_vs_brute_force(seed):
    rng = np.random.default_rng(seed)
    C = int(rng.integers(1, 5))
    L = int(rng.integers(1, 6))
    S = int(rng.integers(2, 11))
    f = rng.integers(1, 50, C)
    b = rng.integers(1, 90, C)
    a = rng.integers(1, 200, C)
    cands = oracle.mem_candidates(f, b, a, layers=L, S=S)
    combos = set()
    for asg in itertools.product(range(C), repeat=L):
        combos.add((int(sum(f[c] for c in asg)), int(sum(b[c] for c in asg)), int(sum(a[c] for c in asg))))
    assert 1 <= len(cands) <= S
    for x in cands:
        assert x in combos
    lat = [fx + bx for fx, bx, _ in cands]
    mem = [mx for _, _, mx in cands]
    assert all(mem[i] < mem[i + 1] and lat[i] > lat[i + 1] for i in range(len(cands) - 1))
    fastest = min(combos, key=lambda x: (x[0] + x[1], x[2], x[0]))
    smallest = min(combos, key=lambda x: (x[2], x[0] + x[1], x[0]))
    assert cands[-1][0] + cands[-1][1] == fastest[0] + fastest[1] and cands[-1][2] == fastest[2]
    assert cands[0][2] == smallest[2] and cands[0][0] + cands[0][1] == smallest[0] + smallest[1]
    if S > 2 and fastest[2] > smallest[2]:
        width = -(-(fastest[2] - smallest[2]) // (S - 2))
        for fx, bx, mx in combos:
            assert any(cf + cb <= fx + bx and cm <= mx + width for cf, cb, cm in cands)


def _one_pair_problem(budget_kib):
    md = Module("m", 1, 1, 1, 1, 0, *H.table(1, {1: (4, 6, 8 * GB, 0)}))
    pb = Problem("pair", 1, 1, [md], np.array([0, 1], np.uint32), np.ones(1, np.uint16),
                 np.array([budget_kib], np.uint32))
    menu = (np.array([[0, 4], [0, 2]], np.uint32), np.array([[0, 6], [0, 4]], np.uint32),
            np.array([[0, 8 * GB], [0, 12 * GB]], np.uint32))
    cs = H.candidates_from_orders(pb, [[1]], [[[("F", 0), ("B", 0)]]])
    return pb, menu, cs


@pytest.mark.parametrize("budget_gb,want_sel,want_mk", [(10, 0, 10), (12, 1, 6), (11, 0, 10)])
def test_selection_spec_one_pair(budget_gb, want_sel, want_mk):
    pb, menu, cs = _one_pair_problem(budget_gb * GB)
    sel, r = oracle.memopt(pb, cs, menu, S=10)
    assert r.status[0] == oracle.ST_OK
    assert sel[0, 0, 0, 0] == want_sel and sel[0, 0, 1, 0] == want_sel
    assert int(r.makespan[0]) == want_mk
    assert int(r.peaks[0, 0]) == (8 if want_sel == 0 else 12) * GB


def _fastest_problem(pb, menu):
    """the same problem with every module's tables replaced by the fastest per-layer strategy"""
    import copy
    f, b, a = menu
    pb2 = copy.deepcopy(pb)
    off = problem_arrays(pb)["tab_off"]
    for i, md in enumerate(pb2.modules):
        sl = slice(int(off[i]), int(off[i + 1]))
        c = int(np.argmin(f[:, sl].astype(np.int64).sum(1) + b[:, sl].astype(np.int64).sum(1)))
        md.f_ns, md.b_ns, md.act_kib = f[c, sl].copy(), b[c, sl].copy(), a[c, sl].copy()
    return pb2


@pytest.mark.parametrize("name", ["toy", "12B"])
def test_unbounded_memory_selects_fastest(name):
    import copy
    pb = copy.deepcopy(gen.make_problem(name))
    pb.budget_kib = np.full(pb.P, (1 << 32) - 1, np.uint32)
    menu = strategy_menu(pb)
    cs = gen.generate(pb, 0, 6, mode=1 if name == "toy" else 0, p_mutate=0, p_bad=0)
    sel, r = oracle.memopt(pb, cs, menu, S=10, threads=4)
    ref = oracle.evaluate(_fastest_problem(pb, menu), cs, threads=4)
    assert np.array_equal(r.status, ref.status)
    ok = r.status == oracle.ST_OK
    assert ok.any()
    assert np.array_equal(r.makespan[ok], ref.makespan[ok])
    assert np.array_equal(r.peaks[ok], ref.peaks[ok])


def test_candidate_zero_everywhere_is_the_fixed_order_oracle():
    # a budget of zero makes every upgrade infeasible (and the base schedule OOM): M4 with
    # candidate 0 must then be exactly O1-O10 on the base tables
    import copy
    pb = copy.deepcopy(gen.make_problem("12B"))
    pb.budget_kib = np.zeros(pb.P, np.uint32)
    cs = gen.generate(pb, 0, 8, p_mutate=0.3, p_bad=0.2)
    sel, r = oracle.memopt(pb, cs, strategy_menu(pb), S=10, threads=4)
    ref = oracle.evaluate(pb, cs, threads=4)
    assert not sel.any()
    for k in ("status", "makespan", "oom_mask", "peaks", "busy"):
        assert np.array_equal(getattr(r, k), getattr(ref, k)), k


def _pairs(pb, cs, x, menu, S):
    """independent per-rank pair data: (F slot, B slot, candidate list) for forward position p"""
    n = int(cs.n[x])
    nm = pb.nmod
    split = cs.split[x].reshape(pb.m, nm)
    dec = pb.seg_decode()
    off = problem_arrays(pb)["tab_off"]
    f, b, a = menu
    out = []
    for r in range(pb.P):
        bits = [(int(cs.fb[x, r, t >> 5]) >> (t & 31)) & 1 for t in range(2 * n)]
        fslots = [t for t in range(2 * n) if not bits[t]]
        bslots = [t for t in range(2 * n) if bits[t]]
        bslot_of = {int(cs.bwd[x, q]): bslots[q] for q in range(n)}
        rows = []
        for p in range(n):
            s = int(cs.fwd[x, p])
            bb, i, j, k = (int(v) for v in dec[s])
            sizes = oracle.split_sizes(int(pb.n_inst()[bb, i]), int(split[bb, i]))
            lo = int(pb.inst_off[bb * nm + i]) + sum(sizes[:j])
            W = int(pb.inst_units[lo:lo + sizes[j]].astype(np.int64).sum())
            md = pb.modules[i]
            lay = int(md.chunk_layers[k * pb.P + r]) if md.chunk_layers is not None else \
                oracle.chunk_layers(md.L, pb.P, md.K)[k * pb.P + r]
            t = int(off[i]) + W
            cl = oracle.mem_candidates(f[:, t], b[:, t], a[:, t], lay, S)
            rows.append((fslots[p], bslot_of[s], cl))
        out.append((fslots, rows))
    return out


@pytest.mark.parametrize("name,count", [("toy", 16), ("12B", 6), ("T2V", 3)])
def test_selection_feasible_and_within_gap(name, count):
    """generated schedules: the selection fits every forward slot (independent re-check), its peak is
    the reported one, the solver's root bound certifies the warm start here, and then the warm start
    is terminated: no single pair can still move up"""
    pb = gen.make_problem(name)
    menu = strategy_menu(pb)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0, p_bad=0)
    base = oracle.evaluate(pb, cs, threads=4)
    sel, r, st = oracle.memopt(pb, cs, menu, S=10, threads=4, stats=True)
    moved = 0
    for x in range(count):
        if base.status[x] != oracle.ST_OK:
            continue
        assert r.status[x] == oracle.ST_OK
        for rk, (fslots, rows) in enumerate(_pairs(pb, cs, x, menu, 10)):
            bud = int(pb.budget_kib[rk])
            cur = [int(sel[x, rk, 0, p]) for p in range(len(rows))]
            moved += sum(cur)

            def used(pt, cur):
                return sum(cl[c][2] for (fs, bs, cl), c in zip(rows, cur) if fs <= pt < bs)
            peak = max(used(pt, cur) for pt in fslots)
            assert peak <= bud
            assert peak == int(r.peaks[x, rk])
            warm, bound, final, nodes, flags = (int(v) for v in st[x, rk])
            assert final == sum(cl[c][0] + cl[c][1] for (_, _, cl), c in zip(rows, cur))
            assert flags == 2 and 1000 * bound >= 950 * final
            for p, (fs, bs, cl) in enumerate(rows):       # termination: no pair can still move up
                if cur[p] + 1 < len(cl):
                    up = list(cur)
                    up[p] += 1
                    assert any(used(pt, up) > bud for pt in fslots if fs <= pt < bs)
    if name != "toy":
        assert moved > 0


@pytest.mark.parametrize("name,x", [("12B", 18), ("12B", 39), ("94B", 3)])
def test_selection_against_highs_at_full_size(name, x):
    """M3 at real size against an independent ILP solver (scipy's HiGHS branch and cut on the
    P:572-582 formulation, solved to a 0.1 % gap): our selection is within 5 % of HiGHS's proven
    lower bound (so of the optimum), and our bound never exceeds HiGHS's feasible optimum"""
    sp = pytest.importorskip("scipy.optimize")
    pb = gen.make_problem(name)
    menu = strategy_menu(pb)
    cs = gen.generate(pb, x, 1, p_mutate=0, p_bad=0)
    sel, r, st = oracle.memopt(pb, cs, menu, S=10, stats=True)
    checked = 0
    for rk, (fslots, rows) in enumerate(_pairs(pb, cs, 0, menu, 10)):
        if rk % max(1, pb.P // 4):
            continue
        bud = int(pb.budget_kib[rk])
        n = len(rows)
        var = [(p, c) for p in range(n) for c in range(len(rows[p][2]))]
        cost = np.array([rows[p][2][c][0] + rows[p][2][c][1] for p, c in var], float)
        A = np.zeros((2 * n, len(var)))
        for v, (p, c) in enumerate(var):
            A[p, v] = 1.0
            for k, pt in enumerate(fslots):
                if rows[p][0] <= pt < rows[p][1]:
                    A[n + k, v] = float(rows[p][2][c][2])
        res = sp.milp(cost, constraints=sp.LinearConstraint(A, [1] * n + [-np.inf] * n, [1] * n + [bud] * n),
                      integrality=np.ones(len(var)), bounds=sp.Bounds(0, 1),
                      options={"mip_rel_gap": 1e-3, "time_limit": 60})
        if res.x is None:
            assert int(st[0, rk, 4]) & 1        # infeasible for HiGHS too: candidate 0 does not fit
            continue
        warm, bound, final, nodes, flags = (int(v) for v in st[0, rk])
        assert 1000 * res.mip_dual_bound >= 950 * final - 1e-6 * final
        assert bound <= res.fun + 1e-6 * res.fun
        checked += 1
    assert checked >= 2


def _tiny_instance(rng):
    P, m = 2, 3
    L = 2 * P                                  # 2 identical layers per chunk
    md = Module("m", L, 1, 1, 3, 0, *H.table(3, {w: (int(rng.integers(2, 9)) * w, int(rng.integers(5, 19)) * w,
                                                     int(rng.integers(2, 6)) * w, 0) for w in (1, 2, 3)}))
    units = rng.integers(1, 4, m).astype(np.uint16)
    pb = Problem("tiny", P, m, [md], np.arange(m + 1, dtype=np.uint32), units, np.zeros(P, np.uint32))
    f0, b0, a0 = md.f_ns.astype(np.int64), md.b_ns.astype(np.int64), md.act_kib.astype(np.int64)
    menu = (np.stack([f0, f0]).astype(np.uint32), np.stack([b0, b0 - (b0 * 2) // 5]).astype(np.uint32),
            np.stack([a0, a0 * 2]).astype(np.uint32))
    orders = H.one_f_one_b(P, m) if rng.random() < 0.5 else H.gpipe(P, m)
    cs = H.candidates_from_orders(pb, [[1] * m], [orders])
    return pb, menu, cs


def _brute(rows, fslots, bud):
    """every selection of a tiny rank (numpy enumeration): (optimum or None, feasible mask, totals)"""
    choices = np.array(list(itertools.product(*[range(len(cl)) for _, _, cl in rows])), np.int64)
    lat = np.stack([np.array([cl[c][0] + cl[c][1] for c in choices[:, p]]) for p, (_, _, cl) in enumerate(rows)], 1)
    mem = np.stack([np.array([cl[c][2] for c in choices[:, p]]) for p, (_, _, cl) in enumerate(rows)], 1)
    live = np.array([[fs <= pt < bs for pt in fslots] for fs, bs, _ in rows], np.int64)   # [pair, point]
    ok = ((mem @ live) <= bud).all(1)
    tot = lat.sum(1)
    return (int(tot[ok].min()) if ok.any() else None), ok, tot, choices


@pytest.mark.parametrize("gap_pm", [50, 0])
def test_selection_gap_against_brute_force(gap_pm):
    """M3 on schedules: the selection is feasible and within the gap of the brute-force
    optimum on EVERY instance ("<= 5%"), exactly optimal with gap 0; the bound never exceeds
    the optimum and the B&B never worsens the warm start."""
    rng = np.random.default_rng(7)
    for trial in range(120):
        pb, menu, cs = _tiny_instance(rng)
        base = oracle.evaluate(pb, cs)
        pk0 = [int(v) for v in base.peaks[0]]
        pb.budget_kib = np.array([int(v * rng.uniform(1.0, 2.2)) for v in pk0], np.uint32)
        sel, r, st = oracle.memopt(pb, cs, menu, S=3, gap_pm=gap_pm, stats=True)
        assert r.status[0] == oracle.ST_OK
        for rk, (fslots, rows) in enumerate(_pairs(pb, cs, 0, menu, 3)):
            best, ok, tot, choices = _brute(rows, fslots, int(pb.budget_kib[rk]))
            got_c = [int(sel[0, rk, 0, p]) for p in range(len(rows))]
            row = np.flatnonzero((choices == np.array(got_c)).all(1))[0]
            assert ok[row]
            got = int(tot[row])
            warm, bound, final, nodes, flags = (int(v) for v in st[0, rk])
            assert final == got and final <= warm and bound <= best <= got
            assert 1000 * best >= (1000 - gap_pm) * got, (trial, rk, best, got)
            assert not flags & 4


def _random_rank(rng, n):
    """a random single-rank order of n stage pairs (forward positions in order, each backward after
    its forward) and Pareto candidate lists (memory up, latency down)"""
    ev = []
    pend = []
    nf = 0
    while nf < n or pend:
        if nf < n and (not pend or rng.random() < 0.55):
            ev.append(("F", nf))
            pend.append(nf)
            nf += 1
        else:
            ev.append(("B", pend.pop(int(rng.integers(len(pend))))))
    sF = [t for t, (d, p) in sorted(enumerate(ev), key=lambda x: x[1][1]) if d == "F"]
    sF = sorted(sF)
    sB = [0] * n
    for t, (d, p) in enumerate(ev):
        if d == "B":
            sB[p] = t
    cands = []
    for p in range(n):
        k = int(rng.integers(1, 5))
        mem = np.cumsum(rng.integers(1, 30, k))
        lat = np.cumsum(rng.integers(1, 40, k))[::-1] + int(rng.integers(20, 200))
        cands.append([(int(lat[c]) - int(lat[c]) // 3, int(lat[c]) // 3, int(mem[c])) for c in range(k)])
    return sF, sB, cands


@pytest.mark.parametrize("gap_pm", [50, 0, 200])
def test_select_rank_against_brute_force(gap_pm):
    """M3 alone on 400 random tiny ranks (n <= 7 pairs, <= 4 candidates): against the brute-force
    optimum -- feasibility, the gap on every instance, exactness at gap 0, the bound never
    above the optimum, the warm start never worsened, infeasibility of candidate 0 reported."""
    rng = np.random.default_rng(1000 + gap_pm)
    searched = 0
    for trial in range(400):
        n = int(rng.integers(1, 8))
        sF, sB, cands = _random_rank(rng, n)
        rows = [(sF[p], sB[p], cands[p]) for p in range(n)]
        live = np.array([[sF[p] <= sF[k] < sB[p] for k in range(n)] for p in range(n)])
        lo = max(sum(cands[p][0][2] for p in range(n) if live[p, k]) for k in range(n))
        hi = max(sum(cands[p][-1][2] for p in range(n) if live[p, k]) for k in range(n))
        bud = int(rng.integers(lo - 3, hi + 2))
        sel, st = oracle.select_rank(sF, sB, cands, bud, gap_pm=gap_pm)
        best, ok, tot, choices = _brute(rows, sF, bud)
        if bud < lo:
            assert st["infeasible"] and sel == [0] * n and best is None
            continue
        row = np.flatnonzero((choices == np.array(sel)).all(1))[0]
        assert ok[row]
        got = int(tot[row])
        assert st["final"] == got <= st["warm"]
        assert st["bound"] <= best
        assert 1000 * best >= (1000 - gap_pm) * got, (trial, best, got, st)
        if gap_pm == 0:
            assert got == best
        assert not st["capped"]
        searched += not st["certified"]
    if gap_pm <= 50:
        assert searched > 10     # the suite does exercise the branch and bound


def test_select_rank_spec_examples():
    # one pair {(10 ms, 8 GB), (6 ms, 12 GB)}: M = 10 GB -> the 8 GB one; M = 12 GB -> 6 ms
    c = [[(10, 0, 8 * GB), (6, 0, 12 * GB)]]
    assert oracle.select_rank([0], [1], c, 10 * GB)[0] == [0]
    assert oracle.select_rank([0], [1], c, 12 * GB)[0] == [1]
    sel, st = oracle.select_rank([0], [1], c, 7 * GB)
    assert st["infeasible"] and sel == [0]


def test_select_rank_greedy_gap_is_closed():
    """a warm start that is > 5 % from the optimum: two pairs live together, room for one upgrade;
    the greedy (best saving per KiB first) takes the small efficient step of pair 0, which blocks
    the large step of pair 1 -- the B&B must find the optimum (pair 1 upgraded)."""
    c = [[(100, 0, 10), (90, 0, 11)],           # saves 10 for 1 KiB (ratio 10)
         [(100, 0, 10), (40, 0, 20)]]           # saves 60 for 10 KiB (ratio 6)
    sel, st = oracle.select_rank([0, 1], [3, 2], c, 30, gap_pm=50)
    assert st["warm"] == 190 and st["final"] == 140 and sel == [0, 1]
    assert not st["certified"] and st["nodes"] > 0
