"""GPU (dip_interleave) vs the oracle's dual-queue greedy (I1-I6): the built
F/B interleavings must be bit-identical, the scores equal, and re-scoring the built records with
dip_eval_schedules must reproduce them (replay identity, App. A.8)."""
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


def fb_rows(pb, m, recs):
    """Test-side reader of the records' word-major F/B rows -> [count, P, fbw]."""
    n_pad = (pb.n_max + 7) // 8 * 8
    nsplit = sum(1 for md in pb.modules if md.max_split > 1)
    off_fwd = (4 + (pb.m * nsplit + 1) // 2 + 15) // 16 * 16
    off_fb = (off_fwd + 4 * n_pad + 15) // 16 * 16
    r = recs.reshape(-1, m.stride)[:, off_fb:off_fb + 4 * pb.fbw * pb.P]
    return np.ascontiguousarray(r).view(np.uint32).reshape(-1, pb.fbw, pb.P).transpose(0, 2, 1)


def run_interleave(pb, cs):
    """dip_interleave (f1) on the GPU, then the built per-rank orders re-scored on the GPU by
    dip_eval_orders (replay)"""
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    s = torch.cuda.current_stream()
    d_rec = torch.from_numpy(m.encode(cs)).cuda()
    d_res = torch.empty(cs.count * 24, dtype=torch.uint8, device="cuda")
    d_pk = torch.empty((cs.count, pb.P), dtype=torch.int32, device="cuda")
    d_ord = torch.empty((cs.count, pb.P, 2 * pb.n_max), dtype=torch.int16, device="cuda")
    dip.interleave(m, ws, d_rec, cs.count, d_res, d_pk, d_orders=d_ord, stream=s)
    win = dip.argmin(m, ws, cs.count, stream=s)
    res = dip.results_view(d_res.cpu().numpy()).copy()
    pk = d_pk.cpu().numpy().view(np.uint32).copy()
    ords = d_ord.cpu().numpy().view(np.uint16).copy()
    d_res2 = torch.empty_like(d_res)
    d_pk2 = torch.empty_like(d_pk)
    dip.eval_orders(m, ws, d_rec, d_ord, cs.count, d_res2, d_pk2, stream=s)
    res2 = dip.results_view(d_res2.cpu().numpy())
    torch.cuda.synchronize()
    return res, pk, ords, win, res2, d_pk2.cpu().numpy().view(np.uint32)


def check(pb, cs):
    res, pk, ords, win, res2, pk2 = run_interleave(pb, cs)
    rords, ref = oracle.interleave(pb, cs, threads=16)
    assert np.array_equal(res["status"], ref.status), np.nonzero(res["status"] != ref.status)[0][:8]
    assert np.array_equal(ords, rords), np.nonzero((ords != rords).any(axis=(1, 2)))[0][:8]
    assert np.array_equal(res["makespan_ns"], ref.makespan)
    assert np.array_equal(res["oom_mask"], ref.oom_mask)
    assert np.array_equal(res["bubble"].view(np.uint64), ref.bubble.view(np.uint64))
    assert np.array_equal(pk.astype(np.uint64), ref.peaks)
    best = oracle.argmin(ref.makespan, ref.status)
    assert win.found == (best >= 0) and (best < 0 or win.global_index == best)
    # replay identity on the GPU: the orders' longest path reproduces the greedy's own times
    for k in ("status", "makespan_ns", "oom_mask"):
        assert np.array_equal(res2[k], res[k]), k
    assert np.array_equal(res2["bubble"].view(np.uint64), res["bubble"].view(np.uint64))
    assert np.array_equal(pk2, pk)
    return res


@pytest.mark.parametrize("name,count", [("toy", 256), ("12B", 512), ("37B", 256), ("T2V", 128), ("94B", 48)])
def test_interleave_parity(name, count):
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0.0, p_bad=0.02)
    check(pb, cs)


def test_interleave_paper_pins_on_gpu():
    # App. A.8: gated with (P - r) activations -> exact 1F1B orders; ungated -> the 1F1B makespan
    for P, m_ in [(4, 8), (8, 16), (3, 5)]:
        pb = H.uniform_problem(P, m_, 1, 2, act=2, budget=[(P - r) * 2 for r in range(P)])
        cs = H.candidates_from_orders(pb, [[1] * m_], [H.one_f_one_b(P, m_)])
        res, pk, ords, win, _, _ = run_interleave(pb, cs)
        assert H.orders_lists(ords[0]) == H.one_f_one_b(P, m_) and int(res["makespan_ns"][0]) == (m_ + P - 1) * 3
    pb = H.uniform_problem(8, 16, 1, 2, act=1)
    cs = H.candidates_from_orders(pb, [[1] * 16], [H.one_f_one_b(8, 16)])
    res, pk, ords, win, _, _ = run_interleave(pb, cs)
    assert pk[0].tolist() == [16, 16, 16, 15, 14, 10, 6, 2]
    # the hand-worked two-rank trace of tests/test_oracle_interleave.py (priorities order the ready set)
    pb = H.uniform_problem(2, 2, 1, 2)
    cs = H.candidates_from_orders(pb, [[1, 1]], [[[("F", 0), ("F", 1), ("B", 1), ("B", 0)]] * 2])
    res, pk, ords, win, _, _ = run_interleave(pb, cs)
    assert H.orders_lists(ords[0]) == [[("F", 0), ("F", 1), ("B", 0), ("B", 1)],
                                       [("F", 0), ("B", 0), ("F", 1), ("B", 1)]]
    assert int(res["makespan_ns"][0]) == 9


def test_interleave_bad_and_non_linear_priorities():
    pb = H.uniform_problem(2, 1, 1, 2, K=2)
    cs = H.candidates_from_orders(pb, [[1]], [[[("F", 0), ("F", 1), ("B", 1), ("B", 0)]] * 2])
    c = cs.subset([0, 0, 0])
    c.fwd[1, :2] = [1, 0]          # not a linear extension: the ready set decides, no deadlock
    c.fwd[2, 1] = c.fwd[2, 0]      # duplicate id -> BAD_ENCODING
    res = check(pb, c)
    assert res["status"].tolist() == [oracle.ST_OK, oracle.ST_OK, oracle.ST_BAD]


@pytest.mark.parametrize("name,count,frac", [("12B", 256, 0.6), ("toy", 512, 0.4), ("94B", 32, 0.7)])
def test_interleave_tight_budgets(name, count, frac):
    # gating and gate lifting at scale (R-30, R-31): budgets at a fraction of the ungated peaks
    # (the kernel's several-ranks-per-step placement must still equal the serial greedy)
    import copy
    pb = copy.deepcopy(gen.make_problem(name))
    cs = gen.generate(pb, 0, count, p_mutate=0.0, p_bad=0.0)
    base = oracle.interleave(pb, cs, threads=16)[1]
    pb.budget_kib = (np.median(base.peaks, axis=0) * frac).astype(np.uint32)
    res = check(pb, cs)
    assert (res["status"] == oracle.ST_OOM).any()


def test_interleave_bench_size_full():
    # the bench's f1 launch shape: 65,536 94B candidates in one dip_interleave call, EVERY one
    # rebuilt by the oracle's interleaving on all host cores
    import os
    pb = gen.make_problem("94B")
    cs = gen.generate(pb, 0, 65536, threads=os.cpu_count() or 1)
    res, pk, ords, win, res2, pk2 = run_interleave(pb, cs)
    rords, ref = oracle.interleave(pb, cs, threads=os.cpu_count() or 1)
    assert np.array_equal(ords, rords), np.nonzero((ords != rords).any(axis=(1, 2)))[0][:8]
    assert np.array_equal(res["status"], ref.status)
    assert np.array_equal(res["makespan_ns"], ref.makespan)
    assert np.array_equal(res["bubble"].view(np.uint64), ref.bubble.view(np.uint64))
    assert np.array_equal(pk.astype(np.uint64), ref.peaks)
    best = oracle.argmin(ref.makespan, ref.status)
    assert win.found == (best >= 0) and (best < 0 or win.global_index == best)
    print(f"RESULT f1 full batch: 65536 94B candidates, orders / scores identical to the oracle")


def test_interleave_gating_and_gate_lifting_on_gpu():
    # the hand-worked one-rank cases of tests/test_oracle_interleave.py (ungated, gated, gate lifted)
    for budget, order in [(10, "FFBB"), (5, "FBFB"), (4, "FBFB")]:
        pb = H.uniform_problem(1, 2, 1, 2, act=5, budget=[budget])
        cs = H.candidates_from_orders(pb, [[1, 1]], [[[("F", 0), ("F", 1), ("B", 0), ("B", 1)]]])
        res, pk, ords, win, _, _ = run_interleave(pb, cs)
        assert "".join(d for d, _ in H.orders_lists(ords[0])[0]) == order
        check(pb, cs)
