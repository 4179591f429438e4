"""Pins of the oracle's dual-queue interleaving (I1-I6, §5.2).

Expected values: the 1F1B closed form, SURVEY App. A.8's exact-order and peak results (derived
there independently of this code), hand-worked traces (gating, gate lifting, and a two-rank case
where a backward stage of lower priority is ready first: the queues' priorities order their READY
stages, reading R-29), and the replay identity: the greedy places every stage at
max(t_last, t_start), so re-timing its per-rank output orders with the fixed-order simulator
(O1-O10, pinned in test_oracle_pins.py) must reproduce its makespan, peaks and bubble exactly.
"""
import numpy as np
import pytest

import gen
import oracle
from tests import helpers as H

OK, OOM, DL, BAD = oracle.ST_OK, oracle.ST_OOM, oracle.ST_DEADLOCK, oracle.ST_BAD


@pytest.mark.parametrize("tf,tb", [(1, 1), (1, 2), (2, 3)])
def test_ungated_makespan_equals_1f1b(tf, tb):
    # App. A.8: ungated, homogeneous single module -> the 1F1B makespan (m+P-1)(t_f+t_b)
    for P in range(1, 7):
        for m in range(1, 9):
            pb = H.uniform_problem(P, m, tf, tb, act=1)
            cs = H.candidates_from_orders(pb, [[1] * m], [H.one_f_one_b(P, m)])
            ords, r = oracle.interleave(pb, cs)
            assert int(r.makespan[0]) == (m + P - 1) * (tf + tb), (P, m)


def test_ungated_front_loads_forwards():
    # App. A.8: P=8, m=16 (t_f=1, t_b=2) ungated, strict "<" in step 3 (R-26): peaks
    # [16,16,16,15,14,10,6,2] instead of 1F1B's [8,7,...,1] -- the reason for memory gating
    pb = H.uniform_problem(8, 16, 1, 2, act=1)
    cs = H.candidates_from_orders(pb, [[1] * 16], [H.one_f_one_b(8, 16)])
    ords, r = oracle.interleave(pb, cs)
    assert r.peaks[0].tolist() == [16, 16, 16, 15, 14, 10, 6, 2]
    assert int(r.makespan[0]) == (16 + 8 - 1) * 3


@pytest.mark.parametrize("tf,tb", [(1, 1), (1, 2), (2, 3)])
def test_gated_reproduces_exact_1f1b_orders(tf, tb):
    # App. A.8: with capacity (P - r) activations per rank, the gated greedy emits exactly Megatron's
    # 1F1B per-rank orders (R-17) for every P <= 8, m <= 16
    for P in range(1, 9):
        for m in range(1, 17):
            pb = H.uniform_problem(P, m, tf, tb, act=3, budget=[(P - r) * 3 for r in range(P)])
            ref = H.candidates_from_orders(pb, [[1] * m], [H.one_f_one_b(P, m)])
            ords, r = oracle.interleave(pb, ref)
            assert H.orders_lists(ords[0]) == H.one_f_one_b(P, m), (P, m)
            assert r.status[0] == OK and r.peaks[0].tolist() == [min(P - k, m) * 3 for k in range(P)]


@pytest.mark.parametrize("name,count", [("toy", 256), ("12B", 96), ("37B", 48), ("T2V", 32), ("94B", 8)])
def test_replay_identity_on_generated(name, count):
    # the greedy's own times == the longest-path replay of the per-rank orders it emits (App. A.8)
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0.0, p_bad=0.0)
    ords, r = oracle.interleave(pb, cs, threads=8)
    rp = oracle.evaluate(pb, cs, threads=8, orders=ords)
    assert (r.status != DL).all()
    for k in ("status", "makespan", "oom_mask", "peaks", "busy"):
        assert np.array_equal(getattr(r, k), getattr(rp, k)), k
    assert np.array_equal(r.bubble.view(np.uint64), rp.bubble.view(np.uint64))
    # every rank runs each segment exactly once as F and once as B
    for x in range(count):
        n = int(cs.n[x])
        for q in range(pb.P):
            row = [int(v) for v in ords[x, q] if v != 0xFFFF]
            assert len(row) == 2 * n and len(set(row)) == 2 * n


def test_priority_orders_the_ready_stages():
    """P = 2, one module, m = 2, t_f = 1, t_b = 2, ungated; forward priority [0, 1], backward
    priority [1, 0] (B of microbatch 1 first). Worked by hand from P:532-544 with reading R-29:
    rank 0: F0 [0,1) F1 [1,2); rank 1: F0 [1,2); at t = 2 rank 1 has F1 (t_start 2) and B0 (t_start
    2, the loss turnaround) ready and B1 not yet: step 4, equal starts -> the backward, B0 [2,4)
    -- an in-order backward queue would wait for its head B1 instead; then F1 [4,5) and B1 [5,7) on
    rank 1, B0 [4,6) and B1 [7,9) on rank 0: makespan 9."""
    pb = H.uniform_problem(2, 2, 1, 2)
    cs = H.candidates_from_orders(pb, [[1, 1]], [[[("F", 0), ("F", 1), ("B", 1), ("B", 0)]] * 2])
    ords, r = oracle.interleave(pb, cs)
    assert H.orders_lists(ords[0]) == [[("F", 0), ("F", 1), ("B", 0), ("B", 1)],
                                       [("F", 0), ("B", 0), ("F", 1), ("B", 1)]]
    assert int(r.makespan[0]) == 9 and r.status[0] == OK
    st, s0, e0 = oracle.timeline(pb, cs, 0, orders=ords)
    assert s0.tolist() == [[0, 1, 4, 7], [1, 2, 4, 5]] and e0.tolist() == [[1, 2, 6, 9], [2, 4, 5, 7]]


def test_gating_respects_budget_when_feasible():
    # with a budget of one forward activation per rank beyond the 1F1B minimum, no rank exceeds it
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 64, p_mutate=0.0, p_bad=0.0)
    ords, r = oracle.interleave(pb, cs, threads=8)
    ok = r.status == OK
    assert ok.any()
    assert (r.peaks[ok] <= pb.budget_kib[None, :].astype(np.uint64)).all()


def test_bad_priority_orders_and_no_deadlock():
    pb = H.uniform_problem(2, 2, 1, 2)
    cs = H.candidates_from_orders(pb, [[1, 1]], [H.one_f_one_b(2, 2)])
    c = cs.subset([0])
    c.fwd[0, 1] = c.fwd[0, 0]                 # duplicate id -> BAD_ENCODING (R-11)
    ords, r = oracle.interleave(pb, c)
    assert r.status[0] == BAD and int(r.makespan[0]) == 2 ** 64 - 1 and (ords == 0xFFFF).all()
    # a forward priority order that is not a linear extension of the segment DAG (k=1 before k=0):
    # the queue's priority only orders its READY stages (R-29), so nothing blocks -- the same
    # schedule as the linear order (k=0 is the only ready forward at the start)
    pb2 = H.uniform_problem(2, 1, 1, 2, K=2)
    c2 = H.candidates_from_orders(pb2, [[1]], [[[("F", 0), ("F", 1), ("B", 1), ("B", 0)]] * 2])
    o1, r1 = oracle.interleave(pb2, c2)
    c2.fwd[0, :2] = [1, 0]
    o2, r2 = oracle.interleave(pb2, c2)
    assert r2.status[0] == OK and int(r2.makespan[0]) == int(r1.makespan[0]) and np.array_equal(o1, o2)


@pytest.mark.parametrize("budget,order,status,peak", [
    (10, "FFBB", OK, 10),      # ungated: F1 (t_start 0) precedes B0 (t_start t_f): step 4, smallest t_start
    (5, "FBFB", OK, 5),        # gated (R-30): the second forward would exceed the budget
    (4, "FBFB", OOM, 5)])      # every rank blocked by its gate only -> the gate is lifted (R-31)
def test_gating_and_gate_lifting_by_hand(budget, order, status, peak):
    # one rank, two microbatches, t_f = 1, t_b = 2, 5 KiB of activation per forward; worked by hand
    # from P:532-548: step 1 places F0; step 2 compares F1 (t_start 0) and B0 (t_start 1 = end of F0)
    pb = H.uniform_problem(1, 2, 1, 2, act=5, budget=[budget])
    cs = H.candidates_from_orders(pb, [[1, 1]], [[[("F", 0), ("F", 1), ("B", 0), ("B", 1)]]])
    ords, r = oracle.interleave(pb, cs)
    got = "".join(d for d, s in H.orders_lists(ords[0])[0])
    assert got == order
    assert r.status[0] == status and int(r.peaks[0, 0]) == peak
    assert int(r.makespan[0]) == 2 * (1 + 2)


@pytest.mark.parametrize("name,count,mode", [("toy", 256, 1), ("12B", 6, 0)])
def test_against_independent_interleaver(name, count, mode):
    """the oracle's I1-I6 == a second, independently written interleaver (tests/refinterleave.py:
    no ready lists, full re-derivation every step) -- orders, makespan, peaks, OOM"""
    from tests import refinterleave
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, mode=mode, p_mutate=0.0, p_bad=0.0)
    ords, r = oracle.interleave(pb, cs, threads=8)
    for x in range(count):
        ref = refinterleave.interleave(pb, cs, x)
        assert ref is not None
        order, mk, peak, oom = ref
        assert H.orders_lists(ords[x]) == order, x
        assert int(r.makespan[x]) == mk and [int(v) for v in r.peaks[x]] == peak
        assert (r.status[x] == OOM) == oom


def test_against_independent_interleaver_tight_budgets():
    """the same with budgets that force gating and gate lifting (R-30, R-31)"""
    import copy
    from tests import refinterleave
    pb = copy.deepcopy(gen.make_problem("toy"))
    cs = gen.generate(pb, 0, 64, mode=1, p_mutate=0.0, p_bad=0.0)
    base = oracle.interleave(pb, cs)[1]
    pb.budget_kib = (np.median(base.peaks, axis=0) * 0.6).astype(np.uint32)
    ords, r = oracle.interleave(pb, cs, threads=8)
    assert (r.status == OOM).any()
    for x in range(64):
        order, mk, peak, oom = refinterleave.interleave(pb, cs, x)
        assert H.orders_lists(ords[x]) == order, x
        assert int(r.makespan[x]) == mk and [int(v) for v in r.peaks[x]] == peak
