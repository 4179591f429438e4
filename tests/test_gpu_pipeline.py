"""The planner flow of one batch end to end on the GPU (§3.2 steps 3-4): score a
batch of candidate schedules and pick the winner, memory-optimise the best candidates, time the
winner's stages and compile it into per-rank action lists -- every result cross-checked against the
oracle or an independent invariant."""
import numpy as np
import pytest

import gen
import oracle
from gen.problem import strategy_menu

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2504_14145_b200 as dip  # noqa: E402


@pytest.mark.parametrize("name,count", [("12B", 8192), ("T2V", 2048)])
def test_plan_one_batch(name, count):
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, threads=16)
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    s = torch.cuda.current_stream()
    recs = m.encode(cs)
    d_rec = torch.from_numpy(recs).cuda()
    d_res = torch.empty(count * 24, dtype=torch.uint8, device="cuda")
    # 1. score everything, take the winner (§8(a))
    dip.eval_schedules(m, ws, d_rec, count, d_res, None, stream=s)
    win = dip.argmin(m, ws, count, stream=s)
    res = dip.results_view(d_res.cpu().numpy())
    assert win.found and res["status"][win.global_index] == dip.CAND_OK
    ok = res["status"] == dip.CAND_OK
    assert win.makespan_ns == res["makespan_ns"][ok].min()
    ref = oracle.evaluate(pb, cs.subset([win.global_index]))
    assert int(ref.makespan[0]) == win.makespan_ns
    # 2. per-layer memory optimisation of the 64 best feasible candidates (f3): never slower, never OOM
    top = np.argsort(np.where(ok, res["makespan_ns"], np.iinfo(np.uint64).max), kind="stable")[:64]
    sub = cs.subset(top)
    m.set_strategies(strategy_menu(pb), 10)
    d_sub = torch.from_numpy(m.encode(sub)).cuda()
    d_res2 = torch.empty(len(top) * 24, dtype=torch.uint8, device="cuda")
    d_sel = torch.empty(len(top) * pb.P * 2 * pb.n_max, dtype=torch.uint8, device="cuda")
    dip.memopt(m, ws, d_sub, len(top), d_sel, d_res2, None, stream=s)
    win2 = dip.argmin(m, ws, len(top), stream=s)
    res2 = dip.results_view(d_res2.cpu().numpy())
    assert (res2["status"] == dip.CAND_OK).all()
    assert (res2["makespan_ns"] <= res["makespan_ns"][top]).all()
    assert win2.makespan_ns <= win.makespan_ns
    rsel, rref = oracle.memopt(pb, sub.subset([win2.global_index]), strategy_menu(pb), S=10)
    assert int(rref.makespan[0]) == win2.makespan_ns
    # 3. the winner's stage timeline and its per-rank action lists (f4), executed back exactly
    x = int(win.global_index)
    shape = (1, pb.P, 2 * pb.n_max)
    d_s = torch.empty(shape, dtype=torch.int64, device="cuda")
    d_e = torch.empty(shape, dtype=torch.int64, device="cuda")
    d_r1 = torch.empty(24, dtype=torch.uint8, device="cuda")
    rec = recs.reshape(count, m.stride)[x]
    dip.timeline(m, ws, torch.from_numpy(rec.copy()).cuda(), 1, d_r1, d_s, d_e, stream=s)
    S = d_s.cpu().numpy().view(np.uint64)[0]
    E = d_e.cpu().numpy().view(np.uint64)[0]
    assert int(E.max()) == win.makespan_ns
    acts, off, nmsg = dip.compile_plan(m, rec, S, E)
    valid, D = dip.validate_plan(m, rec, acts, off)
    assert valid and np.array_equal(D, S)
    assert nmsg > 0 and len(off) == pb.P + 1


@pytest.mark.parametrize("name,count", [("toy", 256), ("12B", 3000), ("T2V", 700)])
def test_device_encode_and_host_view_pipeline(name, count):
    """§8(b) device-mode encode: byte-identical records to the host encoder; dip_eval_host_view (host
    view -> H2D -> device encode -> score -> results D2H -> argmin) == dip_eval_schedules on the
    host-encoded records, results and winner"""
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0.2, p_bad=0.05)
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m, host_chunk=1024)
    s = torch.cuda.current_stream()
    recs = m.encode(cs)
    d_view = [torch.from_numpy(np.ascontiguousarray(getattr(cs, k))).cuda() for k in ("split", "n", "fwd", "bwd", "fb")]
    d_out = torch.empty(count * m.stride, dtype=torch.uint8, device="cuda")
    dip.encode_device(m, d_view, count, d_out, stream=s)
    assert np.array_equal(d_out.cpu().numpy(), recs)
    d_res = torch.empty(count * 24, dtype=torch.uint8, device="cuda")
    dip.eval_schedules(m, ws, torch.from_numpy(recs).cuda(), count, d_res, None, stream=s)
    win = dip.argmin(m, ws, count, stream=s)
    h_view = [torch.from_numpy(np.ascontiguousarray(getattr(cs, k))).pin_memory() for k in ("split", "n", "fwd", "bwd", "fb")]
    h_res = torch.empty(count * 24, dtype=torch.uint8).pin_memory()
    w2 = dip.eval_host_view(m, ws, h_view, count, h_res, stream=s)
    assert np.array_equal(h_res.numpy(), d_res.cpu().numpy())
    assert (w2.found, w2.global_index, w2.makespan_ns) == (win.found, win.global_index, win.makespan_ns)
