"""Exercises every oracle entry point on small, partly malformed inputs (run under sanitizers by
tests/test_sanitizers.py)."""
import numpy as np, gen, oracle
from gen.problem import strategy_menu
from tests import helpers as H
for name in ["toy", "12B"]:
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, 48, mode=1 if name == "toy" else 0, p_mutate=0.2, p_bad=0.1)
    oracle.evaluate(pb, cs, threads=2)
    ords, _ = oracle.interleave(pb, cs, threads=2)
    oracle.evaluate(pb, cs, threads=2, orders=ords)
    oracle.memopt(pb, cs.subset(range(8)), strategy_menu(pb), S=10, threads=2)
    oracle.memopt(pb, cs.subset(range(8)), strategy_menu(pb), S=10, threads=2, gap_pm=0, node_cap=64,
                  orders=ords[:8], stats=True)
    oracle.search(pb, cs.split[0], seed=1, rounds=3, leaves=3, rollouts=3, menu=strategy_menu(pb))
    oracle.timeline(pb, cs, 0)
pb = H.diamond_problem()
cs = gen.generate(pb, 0, 32, p_mutate=0.2, p_bad=0.1)
oracle.evaluate(pb, cs, threads=2)
oracle.interleave(pb, cs, threads=2)
print(oracle.mem_candidates([4, 4, 3], [9, 6, 5], [2, 8, 11], layers=3, S=5))
print(oracle.select_rank([0, 1, 3], [5, 4, 6], [[(9, 1, 3), (5, 1, 9)], [(7, 2, 2)], [(8, 3, 4), (6, 3, 5), (2, 2, 12)]], 14,
                         gap_pm=0))
print(oracle.mcts_table(3, 1, 6, 2, 2, 2.0, 0.5, [[0.5] * 3, [0.8] * 3, [0.7] * 3])["N"])
print("done")
