"""Pins of the oracle's MCTS segment reordering (S1-S6, §5.1).

* exhaustive budget on a tiny instance -> the brute-force optimum over every class order
  ("exhaustive budget -> ... equal to brute force"), the brute force built here with an
  independent priority -> queue-order builder and the (pinned) oracle interleaving;
* the best-so-far trace never decreases;
* the reported best schedule re-scores to the reported makespan with the fixed-order oracle;
* determinism for a seed;
* the tree policy alone (S4-S6), scored by a table over the first class of a sequence
  (so the random completions do not matter), against hand-worked traces: every node's (parent,
  class, N, s) after 9 single-leaf rounds with alpha = 2, beta = 0.5 (the UCB values of every
  selection are written out below), and after 5 two-leaf rounds (virtual visits, R-35). Swapping
  ln N_x and N_v, ignoring alpha, or selecting before every child exists changes these trees.
"""
import itertools

import numpy as np

import gen
import oracle
from gen import Candidates, Module, Problem
from tests import helpers as H


def tiny_problem():
    # one module, P = 2, three microbatches of different work (so the order matters)
    md = Module("m", 2, 1, 1, 4, 0, *H.table(4, {1: (3, 6, 1, 0), 2: (5, 10, 2, 1), 4: (9, 18, 4, 1)}))
    off = np.arange(4, dtype=np.uint32)
    units = np.array([1, 4, 2], np.uint16)
    return Problem("tiny", 2, 3, [md], off, units, np.full(2, 1 << 20, np.uint32))


def orders_from_sequence(pb, split, seq):
    """Independent builder of S2: class priorities -> forward / backward queue orders."""
    nm = pb.nmod
    base = pb.seg_base()
    classes = [(q, k) for q in range(pb.m * nm) if split[q] for k in range(pb.modules[q % nm].K)]
    C = len(classes)
    Cn = 2 * C
    prio = {c: Cn - 1 - p for p, c in enumerate(seq)}
    segs = []
    for q, k in classes:
        b, i = divmod(q, nm)
        for j in range(int(split[q])):
            segs.append((b, i, j, k, int(base[b, i]) + j * pb.modules[i].K + k))
    out = []
    for d in (0, 1):
        done = set()
        order = []
        while len(order) < len(segs):
            ready = []
            for (b, i, j, k, s) in segs:
                if s in done:
                    continue
                K = pb.modules[i].K
                if d == 0:
                    preds = [s - 1] if k > 0 else [int(base[b, p]) + jj * pb.modules[p].K + pb.modules[p].K - 1
                                                   for p in range(nm) if (pb.modules[i].producer_mask >> p) & 1
                                                   for jj in range(int(split[b * nm + p]))]
                else:
                    preds = [s + 1] if k + 1 < K else [int(base[b, c]) + jj * pb.modules[c].K
                                                       for c in range(nm) if (pb.modules[c].producer_mask >> i) & 1
                                                       for jj in range(int(split[b * nm + c]))]
                if all(p in done for p in preds):
                    cls = classes.index((b * nm + i, k)) + (C if d else 0)
                    ready.append(((Cn - 1 - prio[cls]), j, s))
            pick = min(ready)[2]
            done.add(pick)
            order.append(pick)
        out.append(order)
    return out


def brute_force(pb, split):
    nm = pb.nmod
    C = sum(pb.modules[q % nm].K for q in range(pb.m * nm) if split[q])
    perms = list(itertools.permutations(range(2 * C)))
    cs = Candidates(pb, len(perms))
    n = sum(int(split[q]) * pb.modules[q % nm].K for q in range(pb.m * nm))
    for x, seq in enumerate(perms):
        f, b = orders_from_sequence(pb, split, seq)
        cs.split[x] = split
        cs.n[x] = n
        cs.fwd[x, :n] = f
        cs.bwd[x, :n] = b
    ords, r = oracle.interleave(pb, cs, threads=8)
    md = pb.modules[0]                       # one module, L divisible by P: L / P layers per rank
    LB = (md.L // pb.P) * sum(int(md.f_ns[u]) + int(md.b_ns[u]) for u in pb.inst_units)
    ok = r.status == oracle.ST_OK
    return max(LB / float(mk) for mk in r.makespan[ok]), int(r.makespan[ok].min())


def test_exhaustive_budget_finds_brute_force_optimum():
    pb = tiny_problem()
    split = np.ones(3, np.uint8)
    best_score, best_mk = brute_force(pb, split)
    r = oracle.search(pb, split, seed=11, rounds=150, leaves=2, rollouts=10)
    assert r["makespan"] == best_mk
    assert abs(r["score"] - best_score) == 0.0


def test_trace_monotone_and_best_record_rescores():
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 1, p_mutate=0, p_bad=0)
    r = oracle.search(pb, cs.split[0], seed=3, rounds=12, leaves=4, rollouts=6)
    tr = r["trace"]
    assert (np.diff(tr) >= 0).all() and tr[-1] == r["score"] > 0
    c = cs.subset([0])
    n = int(c.n[0])
    c.fwd[0] = r["fwd"]
    c.bwd[0] = r["bwd"]
    rr = oracle.evaluate(pb, c, orders=r["orders"][None])
    assert rr.status[0] == oracle.ST_OK and int(rr.makespan[0]) == r["makespan"]
    assert sorted(r["fwd"][:n].tolist()) == sorted(cs.fwd[0][:n].tolist())


def test_search_is_deterministic_per_seed():
    pb = gen.make_problem("toy")
    cs = gen.generate(pb, 0, 1, mode=1)
    a = oracle.search(pb, cs.split[0], seed=5, rounds=10, leaves=3, rollouts=4)
    b = oracle.search(pb, cs.split[0], seed=5, rounds=10, leaves=3, rollouts=4)
    assert np.array_equal(a["trace"], b["trace"]) and a["makespan"] == b["makespan"]
    assert np.array_equal(a["orders"], b["orders"])


def test_exhaustive_budget_with_chunk_classes():
    # K = 2 chunks per segment: each (microbatch, chunk) is its own class (R-32), so an
    # interleaved-VPP-like order (chunk 0 of both microbatches before chunk 1) is reachable
    md = Module("m", 4, 2, 1, 4, 0, *H.table(4, {1: (3, 6, 1, 0), 3: (7, 14, 3, 1)}))
    pb = Problem("tiny2", 2, 2, [md], np.arange(3, dtype=np.uint32), np.array([1, 3], np.uint16),
                 np.full(2, 1 << 20, np.uint32))
    split = np.ones(2, np.uint8)
    best_score, best_mk = brute_force(pb, split)
    r = oracle.search(pb, split, seed=2, rounds=1200, leaves=100, rollouts=2)
    assert r["makespan"] == best_mk
    assert abs(r["score"] - best_score) == 0.0


def test_search_with_memopt_rescores_and_improves_scores():
    # S3 with M1-M4: the best schedule re-scores through the memory optimisation to the
    # reported makespan; and a rollout never scores lower than without it (pairs only move to
    # faster candidates, and the longest path is monotone in stage latency), so the first round,
    # whose rollouts are the same in both searches, has a best score at least as high
    from gen.problem import strategy_menu
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 1, p_mutate=0, p_bad=0)
    menu = strategy_menu(pb)
    a = oracle.search(pb, cs.split[0], seed=3, rounds=6, leaves=4, rollouts=5)
    b = oracle.search(pb, cs.split[0], seed=3, rounds=6, leaves=4, rollouts=5, menu=menu, S=10)
    c = cs.subset([0])
    c.fwd[0] = b["fwd"]
    c.bwd[0] = b["bwd"]
    sel, rr = oracle.memopt(pb, c, menu, S=10, orders=b["orders"][None])
    assert rr.status[0] == oracle.ST_OK and int(rr.makespan[0]) == b["makespan"]
    assert (np.diff(b["trace"]) >= 0).all()
    assert b["trace"][0] >= a["trace"][0] > 0


def _tree(t):
    return [(int(p), int(c), int(n), round(float(v), 4)) for p, c, n, v in zip(t["parent"], t["cls"], t["N"], t["s"])]


def test_tree_policy_hand_worked_single_leaf():
    """Cn = 3 classes, rollout score = a[first class] with a = (0.5, 0.8, 0.72); alpha = 2, beta =
    0.5, one leaf per round. Rounds 1-3 expand the root's children (0), (1), (2) (unvisited children
    first). Then UCB = s^2 + 0.5 sqrt(ln N_x / N_v):
      r4  root N=3: (0) .25+.5241=.7741  (1) .64+.5241=1.1641  (2) .5184+.5241=1.0425 -> (1), expand (1,0)
      r5  root N=4: .8387, .64+.4163=1.0563, .5184+.5887=1.1071 -> (2), expand (2,0)
      r6  root N=5: .8843, .64+.4485=1.0885, .5184+.4485=.9669 -> (1), expand (1,2)
      r7  root N=6: .9193, .64+.3864=1.0264, .9917 -> (1) [full]: (1,0) and (1,2) both 1.1641, tie
          -> the first, (1,0); expand (1,0,2)
      r8  root N=7: .9475, .9887, .5184+.4932=1.0116 -> (2), expand (2,1)
      r9  root N=8: .9710, .64+.3605=1.0005, .9347 -> (1): (1,0) N=2 1.0563, (1,2) N=1 1.2287 -> (1,2),
          expand (1,2,0)
    Backpropagation: s = max, N + 1 along the path."""
    t = oracle.mcts_table(3, seed=1, rounds=9, leaves=1, rollouts=3, alpha=2.0, beta=0.5,
                          table=[[0.5] * 3, [0.8] * 3, [0.72] * 3])
    assert _tree(t) == [(-1, -1, 9, 0.8), (0, 0, 1, 0.5), (0, 1, 5, 0.8), (0, 2, 3, 0.72), (2, 0, 2, 0.8),
                        (3, 0, 1, 0.72), (2, 2, 2, 0.8), (4, 2, 1, 0.8), (3, 1, 1, 0.72), (6, 0, 1, 0.8)]
    assert t["leaves"][:, 0].tolist() == list(range(1, 10))
    assert t["trace"].tolist() == [0.5] + [0.8] * 8


def test_tree_policy_hand_worked_two_leaves():
    """the same scores, two leaves per round: the first leaf's path carries a virtual visit while
    the second is selected (R-35), so a just-expanded child has N_v = 1 and s = 0 until the round
    is scored (worked with the same UCB as above)"""
    t = oracle.mcts_table(3, seed=1, rounds=5, leaves=2, rollouts=3, alpha=2.0, beta=0.5,
                          table=[[0.5] * 3, [0.8] * 3, [0.72] * 3])
    assert _tree(t) == [(-1, -1, 10, 0.8), (0, 0, 2, 0.5), (0, 1, 5, 0.8), (0, 2, 3, 0.72), (2, 0, 2, 0.8),
                        (3, 0, 1, 0.72), (2, 2, 2, 0.8), (4, 2, 1, 0.8), (3, 1, 1, 0.72), (6, 0, 1, 0.8),
                        (1, 1, 1, 0.5)]


def test_tree_policy_deeper_scores():
    """scores that depend on the first two classes, every completion of a depth-2 prefix scoring the
    same: table[a][b]; the best complete order (2, 0, 1) = 0.9 is found and the root's s is the
    maximum over the table entries reachable"""
    tab = [[0.1, 0.1, 0.2], [0.3, 0.3, 0.4], [0.9, 0.5, 0.5]]
    t = oracle.mcts_table(3, seed=4, rounds=40, leaves=1, rollouts=1, alpha=1.0, beta=0.3, table=tab)
    assert t["trace"][-1] == 0.9 and (np.diff(t["trace"]) >= 0).all()
    # every node's s is the best score seen below it: a node's s >= each child's s
    tr = _tree(t)
    for x, (p, c, n, v) in enumerate(tr):
        if p >= 0:
            assert tr[p][3] >= v and tr[p][2] >= n


def _path(t, v):
    out = []
    while v > 0:
        out.append(int(t["cls"][v]))
        v = int(t["parent"][v])
    return tuple(out[::-1])


def test_depth_first_policy_is_pre_order():
    """P:963-972's DFS variant: the leaves follow a pre-order traversal of the sequence tree with
    children in class order (written out by hand for Cn = 3)"""
    t = oracle.mcts_table(3, seed=1, rounds=13, leaves=1, rollouts=2, alpha=1.0, beta=0.5,
                          table=[[0.5] * 3, [0.8] * 3, [0.7] * 3], policy=2)
    assert [_path(t, int(v)) for v in t["leaves"][:, 0]] == [
        (0,), (0, 1), (0, 1, 2), (0, 2), (0, 2, 1), (1,), (1, 0), (1, 0, 2), (1, 2), (1, 2, 0), (2,), (2, 0), (2, 0, 1)]


def test_random_policy_never_builds_a_tree():
    """P:963-972's random-exploration variant: every rollout is a uniformly random sequence from the
    root; the root is the only node and counts every leaf slot"""
    t = oracle.mcts_table(3, seed=1, rounds=5, leaves=2, rollouts=2, alpha=1.0, beta=0.5,
                          table=[[0.5] * 3, [0.8] * 3, [0.7] * 3], policy=1)
    assert t["leaves"].tolist() == [[0, 0]] * 5 and t["N"].tolist() == [10] and len(t["parent"]) == 1


def test_policies_share_the_rollout_stream():
    """the three policies draw the same rollout counter stream: at equal budget the random policy's
    best is the best of the same number of uniformly random sequences, never above the exhaustive
    optimum, and MCTS's exhaustive-budget optimum is reached"""
    pb = tiny_problem()
    split = np.ones(3, np.uint8)
    best_score, best_mk = brute_force(pb, split)
    for pol in (1, 2):
        r = oracle.search(pb, split, seed=11, rounds=40, leaves=2, rollouts=4, policy=pol)
        assert r["score"] <= best_score and r["makespan"] >= best_mk and (np.diff(r["trace"]) >= 0).all()
