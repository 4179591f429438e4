"""dip_timeline (per-stage start / end on the GPU) vs the oracle's Kahn timeline, and f4 plans
compiled from the GPU timeline execute back to it."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2504_14145_b200 as dip  # noqa: E402


@pytest.mark.parametrize("name,count", [("toy", 64), ("12B", 32), ("T2V", 8), ("94B", 4)])
def test_timeline_matches_oracle_and_plans_round_trip(name, count):
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0.1, p_bad=0.0)
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    recs = m.encode(cs)
    d_rec = torch.from_numpy(recs).cuda()
    d_res = torch.empty(count * 24, dtype=torch.uint8, device="cuda")
    shape = (count, pb.P, 2 * pb.n_max)
    d_s = torch.empty(shape, dtype=torch.int64, device="cuda")
    d_e = torch.empty(shape, dtype=torch.int64, device="cuda")
    dip.timeline(m, ws, d_rec, count, d_res, d_s, d_e, stream=torch.cuda.current_stream())
    S = d_s.cpu().numpy().view(np.uint64)
    E = d_e.cpu().numpy().view(np.uint64)
    res = dip.results_view(d_res.cpu().numpy())
    checked = 0
    for x in range(count):
        st, s, e = oracle.timeline(pb, cs, x)
        assert int(res["status"][x]) == st
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
