"""Exercises every oracle entry point on small, partly malformed inputs (run under sanitizers by
tests/test_sanitizers.py)."""
import numpy as np, gen, oracle
from gen.problem import strategy_menu
from tests import helpers as H
for name in ["toy", "12B"]:
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, 48, mode=1 if name == "toy" else 0, p_mutate=0.2, p_bad=0.1)
    oracle.evaluate(pb, cs, threads=2)
    oracle.interleave(pb, cs, threads=2)
    oracle.memopt(pb, cs.subset(range(8)), strategy_menu(pb), S=10, threads=2)
    oracle.search(pb, cs.split[0], seed=1, rounds=3, leaves=3, rollouts=3, menu=strategy_menu(pb))
    oracle.timeline(pb, cs, 0)
pb = H.diamond_problem()
cs = gen.generate(pb, 0, 32, p_mutate=0.2, p_bad=0.1)
oracle.evaluate(pb, cs, threads=2)
oracle.interleave(pb, cs, threads=2)
print(oracle.mem_candidates([4, 4, 3], [9, 6, 5], [2, 8, 11], layers=3, S=5))
print("done")
