"""Pins of the oracle's per-layer memory optimisation (M1-M4, §5.3).

* M2 candidates: the worked examples of SPEC.md:416-417 ("2 layers x {none: (10 ms, 8 GB),
  checkpoint: (13 ms, 2 GB)}, S=3 -> {(20 ms, 16 GB), (23 ms, 10 GB), (26 ms, 4 GB)}"; "1 layer,
  2 strategies, S=10 -> exactly 2 candidates"), and properties against brute force over every
  per-layer assignment: extremes present, Pareto order, size <= S, and the bucket guarantee
  (every combination is matched by a candidate no slower and at most one bucket width larger);
* M3 selection: SPEC.md:425-426's one-pair examples (M = 10 GB -> the 8 GB candidate, M = 12 GB ->
  the 6 ms one); unbounded memory -> every pair at its fastest candidate, whose re-timed makespan
  equals the fixed-order oracle run on the fastest strategy's tables; on generated schedules an
  independent re-check of feasibility at every forward slot and of the greedy's termination
  (no single pair can still move up); brute force over all selections on tiny instances (the
  greedy is never better than the optimum, and its gap is reported and bounded);
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
def test_selection_feasible_and_greedy_terminated(name, count):
    pb = gen.make_problem(name)
    menu = strategy_menu(pb)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0, p_bad=0)
    base = oracle.evaluate(pb, cs, threads=4)
    sel, r = oracle.memopt(pb, cs, menu, S=10, threads=4)
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
            for p, (fs, bs, cl) in enumerate(rows):       # termination: no pair can still move up
                if cur[p] + 1 < len(cl):
                    up = list(cur)
                    up[p] += 1
                    assert any(used(pt, up) > bud for pt in fslots if fs <= pt < bs)
    if name != "toy":
        assert moved > 0


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


def test_greedy_against_brute_force_optimum():
    rng = np.random.default_rng(7)
    gaps = []
    for trial in range(120):
        pb, menu, cs = _tiny_instance(rng)
        # budget: between the base peak and the all-fastest peak
        base = oracle.evaluate(pb, cs)
        pk0 = [int(v) for v in base.peaks[0]]
        pb.budget_kib = np.array([int(v * rng.uniform(1.0, 2.2)) for v in pk0], np.uint32)
        sel, r = oracle.memopt(pb, cs, menu, S=3)
        assert r.status[0] == oracle.ST_OK
        for rk, (fslots, rows) in enumerate(_pairs(pb, cs, 0, menu, 3)):
            bud = int(pb.budget_kib[rk])
            best = None
            for choice in itertools.product(*[range(len(cl)) for _, _, cl in rows]):
                if all(sum(cl[c][2] for (fs, bs, cl), c in zip(rows, choice) if fs <= pt < bs) <= bud for pt in fslots):
                    tot = sum(cl[c][0] + cl[c][1] for (_, _, cl), c in zip(rows, choice))
                    best = tot if best is None else min(best, tot)
            got = sum(cl[int(sel[0, rk, 0, p])][0] + cl[int(sel[0, rk, 0, p])][1] for p, (_, _, cl) in enumerate(rows))
            assert best is not None and got >= best
            gaps.append(got / best - 1.0)
    gaps = np.array(gaps)
    # the paper accepts a <= 5 % gap from its ILP; the greedy warm start alone meets it on
    # most instances of this suite and stays within 15 % on all of them
    assert (gaps <= 0.05).mean() >= 0.9, np.sort(gaps)[-10:]
    assert gaps.max() <= 0.15, gaps.max()
