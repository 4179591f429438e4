"""Oracle invariants on generated (multi-module) candidates, and agreement with the
independent evaluator in tests/refsim.py (recursive longest path + DFS cycle check)."""
import copy

import numpy as np
import pytest

import gen
import oracle
from tests import refsim

OK, OOM, DL, BAD = oracle.ST_OK, oracle.ST_OOM, oracle.ST_DEADLOCK, oracle.ST_BAD


def _agree(pb, cs, r, idx):
    for x in idx:
        st, mk, pk, bub, busy = refsim.evaluate(pb, cs, int(x))
        assert int(r.status[x]) == st, x
        if st in (OK, OOM):
            assert int(r.makespan[x]) == mk and r.bubble[x] == bub and int(r.busy[x]) == busy, x
        if st != BAD:
            assert r.peaks[x].tolist() == pk, x


def test_toy_all_256_agree_with_independent_evaluator():
    pb = gen.make_problem("toy")
    cs = gen.generate(pb, 0, 256, mode=1)
    r = oracle.evaluate(pb, cs, threads=4)
    _agree(pb, cs, r, range(256))
    assert (r.status == OK).sum() > 200


@pytest.mark.parametrize("name,count", [("12B", 40), ("37B", 24), ("T2V", 16)])
def test_generated_agree_with_independent_evaluator(name, count):
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, p_mutate=0.3, p_bad=0.1)
    r = oracle.evaluate(pb, cs, threads=4)
    _agree(pb, cs, r, range(count))


def test_threads_do_not_change_results():
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 64)
    a = oracle.evaluate(pb, cs, threads=1)
    b = oracle.evaluate(pb, cs, threads=7)
    for k in ("makespan", "status", "oom_mask", "peaks", "busy"):
        assert np.array_equal(getattr(a, k), getattr(b, k))
    assert np.array_equal(a.bubble.view(np.uint64), b.bubble.view(np.uint64))


def test_single_rank_has_no_bubble():
    # P = 1: every edge is same-rank, makespan = sum of latencies, bubble = 0 (P:248 definition)
    pb = gen.make_problem("toy")
    pb1 = copy.deepcopy(pb)
    pb1.P = 1
    pb1.budget_kib = pb.budget_kib[:1].copy()
    cs = gen.generate(pb1, 0, 64, mode=1)
    r = oracle.evaluate(pb1, cs)
    ok = r.status == OK
    assert ok.all()
    assert np.array_equal(r.makespan, r.busy) and (r.bubble == 0.0).all()


def test_makespan_lower_bound_and_monotone_in_latency():
    pb = gen.make_problem("37B")
    cs = gen.generate(pb, 0, 48)
    r = oracle.evaluate(pb, cs, threads=4)
    timed = (r.status == OK) | (r.status == OOM)
    assert timed.sum() > 30
    # makespan >= busy / P (the busiest rank is at least the mean)
    assert (r.makespan[timed] * pb.P >= r.busy[timed]).all()
    pb2 = copy.deepcopy(pb)
    for md in pb2.modules:
        md.b_ns = md.b_ns + (md.b_ns > 0).astype(np.uint32) * 1000
    r2 = oracle.evaluate(pb2, cs, threads=4)
    assert np.array_equal(r.status == DL, r2.status == DL)
    assert (r2.makespan[timed] > r.makespan[timed]).all()
    assert np.array_equal(r.peaks, r2.peaks)        # memory depends on order only (R-9)


def test_generator_statuses_mostly_timed():
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 400)
    r = oracle.evaluate(pb, cs, threads=8)
    timed = ((r.status == OK) | (r.status == OOM)).mean()
    assert timed >= 0.9
    assert (r.status == BAD).sum() == ((cs.family >> 6) & 1).sum() or (r.status == BAD).sum() > 0


def test_diamond_modules_agree_with_independent_evaluator():
    # four modules in a diamond (two producer modules joined by a K = 2 fusion module feeding a
    # K = 2 LLM), split sub-microbatches on both sides of each join, microbatches without vision
    from tests import helpers as H
    pb = H.diamond_problem()
    cs = gen.generate(pb, 0, 120, p_mutate=0.1, p_bad=0.05)
    r = oracle.evaluate(pb, cs, threads=4)
    _agree(pb, cs, r, range(120))
    hist = np.bincount(r.status, minlength=4)
    assert hist[OK] > 0 and hist[OOM] > 0 and hist[DL] > 0 and hist[BAD] > 0
