"""The f1 kernel places on several ranks per step (csrc/dip_order.cu, BUILD: a conservative
lookahead over the ring of ranks). tests/lookahead_model.py restates that step rule in Python; here
it must reproduce the serial greedy of P:526-548 exactly -- whose orders must in turn be the
oracle's -- including budgets that gate forwards and force the relaxed step (R-30, R-31), uniform
pipelines with zero p2p (no lookahead at all) and two / three ranks (the ring's corner cases).
The GPU kernel itself is held to the oracle by tests/test_gpu_interleave.py."""
import copy

import numpy as np
import pytest

import gen
import oracle
from tests import helpers as H
from tests import lookahead_model as LM


def test_model_serial_is_the_oracle():
    pb = gen.make_problem("toy")
    cs = gen.generate(pb, 0, 16, mode=1, p_mutate=0.0, p_bad=0.0)
    ords, _ = oracle.interleave(pb, cs)
    for x in range(16):
        sim = LM.Sim(LM.build(pb, cs, x))
        sim.run(False)
        assert sim.order == H.orders_lists(ords[x]), x


@pytest.mark.parametrize("mode", [0, 1])
def test_parallel_steps_equal_serial_toy(mode):
    pb = gen.make_problem("toy")
    cs = gen.generate(pb, 0, 48, mode=mode, p_mutate=0.0, p_bad=0.0)
    tot = [0, 0]
    for x in range(48):
        ns, npar = LM.compare(pb, cs, x)
        tot[0] += ns
        tot[1] += npar
    assert tot[1] < tot[0]          # some steps do place on more than one rank


@pytest.mark.parametrize("frac", [0.6, 0.4])
def test_parallel_steps_equal_serial_tight_budgets(frac):
    pb = copy.deepcopy(gen.make_problem("toy"))
    cs = gen.generate(pb, 0, 32, mode=1, p_mutate=0.0, p_bad=0.0)
    base = oracle.interleave(pb, cs)[1]
    pb.budget_kib = (np.median(base.peaks, axis=0) * frac).astype(np.uint32)
    gated = 0
    for x in range(32):
        LM.compare(pb, cs, x)
        gated += int(oracle.interleave(pb, cs, x, 1)[1].status[0] == oracle.ST_OOM)
    assert gated > 0


@pytest.mark.parametrize("P,m,p2p,nit", [(2, 4, 0, 3), (3, 5, 1, 3), (4, 6, 0, 1), (5, 7, 2, 8)])
def test_parallel_steps_equal_serial_uniform(P, m, p2p, nit):
    pb = H.uniform_problem(P, m, 2, 3, act=1, p2p=p2p)
    cs = gen.generate(pb, 0, 8, mode=1, p_mutate=0.0, p_bad=0.0)
    for x in range(8):
        LM.compare(pb, cs, x, nit)
