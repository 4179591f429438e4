"""GPU f3 (dip_set_strategies / dip_memopt, §5.3) vs the oracle (M1-M4):
the candidate table of every stage-pair type and width equals oracle.mem_candidates, the per-rank
selections are identical, and the re-timed scores are identical, on every config (generated
schedules incl. mutated / deadlocked / malformed ones), at several S and at the bench batch size
on sampled candidates."""
import numpy as np
import pytest

import gen
import oracle
from gen.problem import problem_arrays, strategy_menu

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2504_14145_b200 as dip  # noqa: E402


def chunk_rows(pb):
    """(module, layers) stage-pair types of the problem"""
    out = set()
    for i, md in enumerate(pb.modules):
        lay = md.chunk_layers if md.chunk_layers is not None else oracle.chunk_layers(md.L, pb.P, md.K)
        for v in lay:
            out.add((i, int(v)))
    return sorted(out)


@pytest.mark.parametrize("name,S", [("toy", 10), ("12B", 10), ("37B", 3), ("T2V", 16), ("94B", 10), ("12B", 2)])
def test_candidate_table_parity(name, S):
    pb = gen.make_problem(name)
    menu = strategy_menu(pb)
    m = dip.Model(pb, 0)
    m.set_strategies(menu, S)
    off = problem_arrays(pb)["tab_off"]
    f, b, a = menu
    for i, lay in chunk_rows(pb):
        for W in range(pb.modules[i].w_max + 1):
            t = int(off[i]) + W
            ref = oracle.mem_candidates(f[:, t], b[:, t], a[:, t], lay, S) if lay else [(0, 0, 0)]
            assert m.strategy_candidates(i, lay, W) == ref, (i, lay, W)


def run(pb, cs, S=10, menu=None, gap_pm=50, node_cap=4096, stats=None):
    m = dip.Model(pb, 0)
    m.set_strategies(strategy_menu(pb) if menu is None else menu, S)
    dip.set_memopt_solver(m, gap_pm, node_cap)
    ws = dip.Workspace(m)
    s = torch.cuda.current_stream()
    d_rec = torch.from_numpy(m.encode(cs)).cuda()
    d_res = torch.empty(cs.count * 24, dtype=torch.uint8, device="cuda")
    d_pk = torch.empty((cs.count, pb.P), dtype=torch.int32, device="cuda")
    d_sel = torch.empty(cs.count * pb.P * 2 * pb.n_max, dtype=torch.uint8, device="cuda")
    dip.memopt(m, ws, d_rec, cs.count, d_sel, d_res, d_pk, stream=s)
    win = dip.argmin(m, ws, cs.count, stream=s)
    torch.cuda.synchronize()
    res = dip.results_view(d_res.cpu().numpy()).copy()
    if stats is not None:
        stats.update(dip.memopt_stats(ws, stream=s))
    return res, d_pk.cpu().numpy().view(np.uint32).copy(), d_sel.cpu().numpy().reshape(cs.count, pb.P, 2, pb.n_max), win


def check(pb, cs, S=10, idx=None, menu=None, gap_pm=50, node_cap=4096):
    """GPU selections, re-timed results and solver counters == the oracle's (M1-M4)"""
    menu = strategy_menu(pb) if menu is None else menu
    gst = {}
    res, pk, sel, win = run(pb, cs, S, menu, gap_pm, node_cap, gst)
    sub = cs if idx is None else cs.subset(idx)
    rsel, ref, rst = oracle.memopt(pb, sub, menu, S=S, threads=16, gap_pm=gap_pm, node_cap=node_cap, stats=True)
    if idx is None and not (ref.status == oracle.ST_BAD).any():
        # the solver's counters over every (record, rank) with n > 0 and a feasible candidate 0 (the
        # selection kernel checks only the record's necessary conditions, so a malformed record the
        # scorer rejects may still be counted there: compared on batches without such records)
        fl = rst[:, :, 4].astype(np.int64)
        solved = (fl & 9) == 0
        want = {"solved": int(solved.sum()), "certified": int((solved & ((fl & 2) > 0)).sum()),
                "searched": int((solved & ((fl & 2) == 0)).sum()), "capped": int(((fl & 4) > 0).sum()),
                "nodes": int(rst[:, :, 3].sum())}
        assert gst == want, (gst, want)
    if idx is not None:
        res, pk, sel = res[idx], pk[idx], sel[idx]
    assert np.array_equal(res["status"], ref.status), np.nonzero(res["status"] != ref.status)[0][:8]
    good = ref.status != oracle.ST_BAD
    assert np.array_equal(sel[good], rsel[good]), np.nonzero((sel != rsel).any(axis=(1, 2, 3)) & good)[0][:8]
    assert np.array_equal(res["makespan_ns"], ref.makespan)
    assert np.array_equal(res["oom_mask"], ref.oom_mask)
    assert np.array_equal(res["bubble"].view(np.uint64), ref.bubble.view(np.uint64))
    assert np.array_equal(pk.astype(np.uint64), ref.peaks)
    if idx is None:
        best = oracle.argmin(ref.makespan, ref.status)
        assert win.found == (best >= 0) and (best < 0 or win.global_index == best)
    return res, sel


@pytest.mark.parametrize("name,count", [("toy", 256), ("12B", 256), ("37B", 96), ("T2V", 64), ("94B", 24)])
def test_memopt_parity(name, count):
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0.04, p_bad=0.02)
    res, sel = check(pb, cs)
    if name != "toy":
        assert sel.any()                       # some pairs moved off candidate 0


@pytest.mark.parametrize("S", [2, 3, 16])
def test_memopt_parity_other_S(S):
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 96, p_mutate=0.04, p_bad=0.02)
    check(pb, cs, S=S)


def test_memopt_bench_size_sampled():
    # the bench's f3 launch shape: 16,384 94B schedules in one call, 1,024 sampled against the oracle
    pb = gen.make_problem("94B")
    cs = gen.generate(pb, 0, 16384, threads=16)
    idx = np.unique(np.concatenate([[0, 1, 2, 4095, 4096, 8191, 16382, 16383],
                                    np.random.default_rng(5).choice(16384, 1016, replace=False)]))
    check(pb, cs, idx=idx)


def _tiny(rng):
    from tests.test_oracle_memopt import _tiny_instance
    pb, menu, cs = _tiny_instance(rng)
    pk0 = [int(v) for v in oracle.evaluate(pb, cs).peaks[0]]
    pb.budget_kib = np.array([int(v * rng.uniform(1.0, 2.2)) for v in pk0], np.uint32)
    return pb, menu, cs


@pytest.mark.parametrize("gap_pm", [50, 0])
def test_memopt_branch_and_bound_tiny(gap_pm):
    """the ILP solver's branch and bound (M3c) on the tiny schedules of the oracle's brute-force pins:
    identical selections, scores and solver counters (children visited included)"""
    rng = np.random.default_rng(7)
    searched = 0
    for trial in range(40):
        pb, menu, cs = _tiny(rng)
        check(pb, cs, S=3, menu=menu, gap_pm=gap_pm)
        st = {}
        run(pb, cs, 3, menu, gap_pm, 4096, st)
        searched += st["searched"]
    assert searched > 0


def test_memopt_branch_and_bound_full_size():
    """exact solving (gap 0) at 12B size runs the depth-first search into its child budget: the GPU
    must walk the oracle's tree node for node (same incumbent, same child count, same stops)"""
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 6, p_mutate=0, p_bad=0)
    check(pb, cs, gap_pm=0, node_cap=200)


def test_strategy_menu_guards():
    import copy
    pb = gen.make_problem("12B")
    f, b, a = strategy_menu(pb)
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    d = torch.zeros(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(dip.DipError) as e:            # no menu yet
        dip.memopt(m, ws, d, 1, d, d, None)
    assert e.value.code == 1
    for S in (1, 17):                                  # S out of range
        with pytest.raises(dip.DipError) as e:
            m.set_strategies((f, b, a), S)
        assert e.value.code == 1
    # (equal-memory / equal-latency candidates cannot survive the pruning -- the fastest, the
    # smallest and every bucket winner break ties the same way -- so that host check is only a
    # safety net and has no reachable input)
    pb2 = copy.deepcopy(pb)                            # budgets beyond the int32 selection
    pb2.budget_kib = np.full(pb.P, (1 << 31) + 5, np.uint32)
    m2 = dip.Model(pb2, 0)
    with pytest.raises(dip.DipError) as e:
        m2.set_strategies((f, b, a), 10)
    assert e.value.code == 4
    m.set_strategies((f, b, a), 10)                    # and a valid menu still loads afterwards
    assert m.strategy_candidates(1, oracle.chunk_layers(pb.modules[1].L, pb.P, pb.modules[1].K)[0], 5)


@pytest.mark.parametrize("name,count", [("toy", 128), ("12B", 128), ("T2V", 32), ("94B", 16)])
def test_memopt_on_interleaved_orders(name, count):
    """f2's rollout: dip_interleave's per-rank orders -> dip_memopt on those orders ->
    re-timing with the selection (dip_eval_orders); selections, scores and peaks == the oracle's
    M1-M4 on the oracle's own interleaving"""
    pb = gen.make_problem(name)
    menu = strategy_menu(pb)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0.0, p_bad=0.02)
    m = dip.Model(pb, 0)
    m.set_strategies(menu, 10)
    ws = dip.Workspace(m)
    s = torch.cuda.current_stream()
    d_rec = torch.from_numpy(m.encode(cs)).cuda()
    d_res = torch.empty(count * 24, dtype=torch.uint8, device="cuda")
    d_pk = torch.empty((count, pb.P), dtype=torch.int32, device="cuda")
    d_ord = torch.empty((count, pb.P, 2 * pb.n_max), dtype=torch.int16, device="cuda")
    d_sel = torch.empty(count * pb.P * 2 * pb.n_max, dtype=torch.uint8, device="cuda")
    dip.interleave(m, ws, d_rec, count, d_res, None, d_orders=d_ord, stream=s)
    dip.memopt(m, ws, d_rec, count, d_sel, d_res, d_pk, stream=s, d_orders=d_ord)
    torch.cuda.synchronize()
    res = dip.results_view(d_res.cpu().numpy()).copy()
    sel = d_sel.cpu().numpy().reshape(count, pb.P, 2, pb.n_max)
    rords, _ = oracle.interleave(pb, cs, threads=16)
    assert np.array_equal(d_ord.cpu().numpy().view(np.uint16), rords)
    rsel, ref = oracle.memopt(pb, cs, menu, S=10, threads=16, orders=rords)
    assert np.array_equal(res["status"], ref.status)
    good = ref.status != oracle.ST_BAD
    assert np.array_equal(sel[good], rsel[good])
    assert np.array_equal(res["makespan_ns"], ref.makespan)
    assert np.array_equal(res["bubble"].view(np.uint64), ref.bubble.view(np.uint64))
    assert np.array_equal(d_pk.cpu().numpy().view(np.uint32).astype(np.uint64), ref.peaks)
    if name != "toy":
        assert sel[good].any()


def test_strategy_menu_raises_the_makespan_bound():
    """a menu whose candidates are slower than the base tables must raise the model's
    makespan bound (the fused argmin key's packing and the 2^53 bubble guard use it), and f3's
    scores stay exact against the oracle with such a menu"""
    pb = gen.make_problem("12B")
    f, b, a = strategy_menu(pb)
    slow = (f.astype(np.int64) * 20).astype(np.uint32), (b.astype(np.int64) * 20).astype(np.uint32), a
    m = dip.Model(pb, 0)
    b0 = m.info["makespan_bound"]
    m.set_strategies(slow, 10)
    assert m.refresh_info()["makespan_bound"] > b0
    cs = gen.generate(pb, 0, 64, p_mutate=0.0, p_bad=0.0)
    check(pb, cs, menu=slow)
