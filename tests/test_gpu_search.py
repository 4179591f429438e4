"""GPU-backed MCTS (dip_search) vs the oracle's MCTS (S1-S6): with the same seed
and budget the two searches must take the same trajectory -- identical best-so-far trace, best
makespan and best schedule -- because every rollout score is bit-exact (f1 parity)."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2504_14145_b200 as dip  # noqa: E402


@pytest.mark.parametrize("name,rounds,leaves,rollouts", [("toy", 30, 4, 6), ("12B", 8, 8, 8), ("T2V", 4, 4, 4),
                                                          ("37B", 4, 6, 5)])
def test_search_matches_oracle_trajectory(name, rounds, leaves, rollouts):
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, 1, mode=1 if name == "toy" else 0, p_mutate=0, p_bad=0)
    split = cs.split[0]
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    g = dip.search(m, ws, split, seed=9, rounds=rounds, leaves=leaves, rollouts=rollouts, alpha=1.0, beta=0.5,
                   stream=torch.cuda.current_stream())
    o = oracle.search(pb, split, seed=9, rounds=rounds, leaves=leaves, rollouts=rollouts, alpha=1.0, beta=0.5)
    assert np.array_equal(g["trace"], o["trace"])
    assert g["makespan"] == o["makespan"] and g["score"] == o["score"]
    assert np.array_equal(g["orders"], o["orders"])
    assert g["scored"] == o["scored"]


@pytest.mark.parametrize("name,rounds,leaves,rollouts", [("toy", 12, 4, 4), ("12B", 6, 8, 6), ("T2V", 3, 4, 3)])
def test_search_with_memopt_matches_oracle_trajectory(name, rounds, leaves, rollouts):
    # every rollout is interleaved (f1) and then memory-optimised (f3) before scoring
    from gen.problem import strategy_menu
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, 1, mode=1 if name == "toy" else 0, p_mutate=0, p_bad=0)
    split = cs.split[0]
    menu = strategy_menu(pb)
    m = dip.Model(pb, 0)
    m.set_strategies(menu, 10)
    ws = dip.Workspace(m)
    g = dip.search(m, ws, split, seed=4, rounds=rounds, leaves=leaves, rollouts=rollouts, alpha=1.0, beta=0.5,
                   stream=torch.cuda.current_stream(), memopt=True)
    o = oracle.search(pb, split, seed=4, rounds=rounds, leaves=leaves, rollouts=rollouts, alpha=1.0, beta=0.5,
                      menu=menu, S=10)
    assert np.array_equal(g["trace"], o["trace"])
    assert g["makespan"] == o["makespan"] and g["score"] == o["score"]
    assert np.array_equal(g["orders"], o["orders"])


def test_search_beats_templates_on_94B_winner_split():
    """on the split of the 94B bench winner, the GPU search (8 rounds x 64 leaves x
    4 rollouts) reaches a makespan no worse than the generator's own template orders run through f1,
    and far below the same orders at fixed order"""
    pb = gen.make_problem("94B")
    cs = gen.generate(pb, 2696, 1)
    fixed = oracle.evaluate(pb, cs)
    _, tf1 = oracle.interleave(pb, cs)
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    g = dip.search(m, ws, cs.split[0], seed=pb.seed, rounds=8, leaves=64, rollouts=4, alpha=1.0, beta=0.5,
                   stream=torch.cuda.current_stream())
    assert g["found"] and g["makespan"] <= int(tf1.makespan[0]) < int(fixed.makespan[0])
    print(f"RESULT f2 94B winner split: search {g['makespan']} ns, template f1 {int(tf1.makespan[0])} ns, "
          f"template fixed order {int(fixed.makespan[0])} ns")


@pytest.mark.parametrize("name,policy", [("toy", 1), ("toy", 2), ("12B", 1), ("12B", 2)])
def test_exploration_policies_match_oracle_trajectory(name, policy):
    """the paper's comparison variants: random exploration and depth-first search take the
    oracle's trajectory exactly (same rollout stream, same scorer)"""
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, 1, mode=1 if name == "toy" else 0, p_mutate=0, p_bad=0)
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    g = dip.search(m, ws, cs.split[0], seed=7, rounds=6, leaves=8, rollouts=4, policy=policy,
                   stream=torch.cuda.current_stream())
    o = oracle.search(pb, cs.split[0], seed=7, rounds=6, leaves=8, rollouts=4, policy=policy)
    assert np.array_equal(g["trace"], o["trace"]) and g["makespan"] == o["makespan"]
    assert np.array_equal(g["orders"], o["orders"]) and g["scored"] == o["scored"]


def test_search_time_budget_stops_early_on_the_same_trajectory():
    """the loop runs until a time budget is exhausted; the rounds it did are a prefix of
    the full search's trajectory"""
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 1, p_mutate=0, p_bad=0)
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    full = dip.search(m, ws, cs.split[0], seed=3, rounds=40, leaves=64, rollouts=4, stream=torch.cuda.current_stream())
    part = dip.search(m, ws, cs.split[0], seed=3, rounds=40, leaves=64, rollouts=4, time_budget_ms=1e-3,
                      stream=torch.cuda.current_stream())
    k = part["rounds_done"]
    assert 1 <= k < 40 and np.array_equal(part["trace"][:k], full["trace"][:k])


def test_search_trajectory_at_94B():
    """the f2 trajectory at the largest config, with and without f3 per rollout"""
    from gen.problem import strategy_menu
    pb = gen.make_problem("94B")
    cs = gen.generate(pb, 2696, 1)
    menu = strategy_menu(pb)
    m = dip.Model(pb, 0)
    m.set_strategies(menu, 10)
    ws = dip.Workspace(m)
    for memopt, (rounds, leaves, rollouts) in ((False, (2, 8, 4)), (True, (1, 4, 2))):
        g = dip.search(m, ws, cs.split[0], seed=5, rounds=rounds, leaves=leaves, rollouts=rollouts, memopt=memopt,
                       stream=torch.cuda.current_stream())
        o = oracle.search(pb, cs.split[0], seed=5, rounds=rounds, leaves=leaves, rollouts=rollouts,
                          menu=menu if memopt else None, S=10)
        assert np.array_equal(g["trace"], o["trace"]) and g["makespan"] == o["makespan"], memopt
        assert np.array_equal(g["orders"], o["orders"])
