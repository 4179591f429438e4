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


@pytest.mark.parametrize("name,count", [("toy", 64), ("12B", 16), ("94B", 2)])
def test_order_timelines_and_plans_of_interleaved_schedules(name, count):
    """schedules built by f1 (per-rank orders): dip_eval_orders' per-slot timelines == the oracle's
    timeline of the same orders, and the f4 plan compiled from them executes back to them"""
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0.0, p_bad=0.0)
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    s = torch.cuda.current_stream()
    recs = m.encode(cs)
    d_rec = torch.from_numpy(recs).cuda()
    d_res = torch.empty(count * 24, dtype=torch.uint8, device="cuda")
    shape = (count, pb.P, 2 * pb.n_max)
    d_ord = torch.empty(shape, dtype=torch.int16, device="cuda")
    dip.interleave(m, ws, d_rec, count, d_res, None, d_orders=d_ord, stream=s)
    d_s = torch.empty(shape, dtype=torch.int64, device="cuda")
    d_e = torch.empty(shape, dtype=torch.int64, device="cuda")
    dip.eval_orders(m, ws, d_rec, d_ord, count, d_res, None, d_start=d_s, d_end=d_e, stream=s)
    torch.cuda.synchronize()
    O = d_ord.cpu().numpy().view(np.uint16)
    S = d_s.cpu().numpy().view(np.uint64)
    E = d_e.cpu().numpy().view(np.uint64)
    for x in range(count):
        st, s0, e0 = oracle.timeline(pb, cs, x, orders=O)
        assert s0 is not None
        n2 = s0.shape[1]
        assert np.array_equal(S[x, :, :n2], s0) and np.array_equal(E[x, :, :n2], e0)
        rec = recs.reshape(count, m.stride)[x]
        acts, off, nmsg = dip.compile_plan(m, rec, S[x], E[x], orders=O[x])
        ok, D = dip.validate_plan(m, rec, acts, off, orders=O[x])
        assert ok and np.array_equal(D, S[x])
