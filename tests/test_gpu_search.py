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
from tests.test_gpu_interleave import fb_rows  # noqa: E402


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
    rec = g["record"]
    n = int(cs.n[0])
    assert np.array_equal(fb_rows(pb, m, rec[None, :])[0], o["bits"])
    assert g["scored"] == rounds * leaves * rollouts or g["scored"] <= rounds * leaves * rollouts


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
    assert np.array_equal(fb_rows(pb, m, g["record"][None, :])[0], o["bits"])
