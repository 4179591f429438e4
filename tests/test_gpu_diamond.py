"""Every GPU entry point on a four-module diamond (vision + audio -> fusion (K = 2) -> LLM (K = 2)):
joins with several producer modules and split sub-microbatches on both sides -- scorer, f1
interleaving, f3 memory optimisation, f2 search and f4 timelines, each against the oracle."""
import numpy as np
import pytest

import gen
import oracle
from tests import helpers as H

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2504_14145_b200 as dip  # noqa: E402
from tests.test_gpu_parity import assert_parity, run_gpu  # noqa: E402
from tests import test_gpu_interleave as TI  # noqa: E402
from tests import test_gpu_memopt as TM  # noqa: E402


@pytest.fixture(scope="module", params=[3, 4, 6])
def diamond(request):
    # P = 3 and 6 leave idle lanes in the G = 4 / 8 lane groups
    pb = H.diamond_problem(P=request.param)
    return pb, gen.generate(pb, 0, 512, p_mutate=0.1, p_bad=0.05)


def test_diamond_scorer(diamond):
    pb, cs = diamond
    res, pk, win = run_gpu(pb, cs)
    assert_parity(pb, cs, res, pk, win)


def test_diamond_interleave(diamond):
    pb, cs = diamond
    TI.check(pb, cs)


def test_diamond_memopt(diamond):
    pb, cs = diamond
    TM.check(pb, cs.subset(range(128)))


def test_diamond_search(diamond):
    pb, cs = diamond
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    g = dip.search(m, ws, cs.split[0], seed=3, rounds=6, leaves=6, rollouts=5, stream=torch.cuda.current_stream())
    o = oracle.search(pb, cs.split[0], seed=3, rounds=6, leaves=6, rollouts=5)
    assert np.array_equal(g["trace"], o["trace"]) and g["makespan"] == o["makespan"]


def test_diamond_timeline_and_plans(diamond):
    pb, cs = diamond
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    count = 16
    recs = m.encode(cs.subset(range(count)))
    shape = (count, pb.P, 2 * pb.n_max)
    d_s = torch.empty(shape, dtype=torch.int64, device="cuda")
    d_e = torch.empty(shape, dtype=torch.int64, device="cuda")
    d_res = torch.empty(count * 24, dtype=torch.uint8, device="cuda")
    dip.timeline(m, ws, torch.from_numpy(recs).cuda(), count, d_res, d_s, d_e, stream=torch.cuda.current_stream())
    S = d_s.cpu().numpy().view(np.uint64)
    E = d_e.cpu().numpy().view(np.uint64)
    checked = 0
    for x in range(count):
        st, s, e = oracle.timeline(pb, cs, x)
        if s is None:
            continue
        n2 = s.shape[1]
        assert np.array_equal(S[x, :, :n2], s) and np.array_equal(E[x, :, :n2], e)
        rec = recs.reshape(count, m.stride)[x]
        acts, off, nmsg = dip.compile_plan(m, rec, S[x], E[x])
        ok, D = dip.validate_plan(m, rec, acts, off)
        assert ok and np.array_equal(D, S[x])
        checked += 1
    assert checked > 0
