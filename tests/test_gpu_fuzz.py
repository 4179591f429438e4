"""Malformed inputs through every GPU entry point: random splits, counts, segment ids (in and out
of range, duplicates, 0xFFFF padding in the wrong places) and random F/B bits. Nothing may crash
or read out of bounds; statuses and results must equal the oracle's (mostly BAD_ENCODING, with
the occasional valid, deadlocked or OOM schedule among near-valid mutations)."""
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
from tests.test_gpu_parity import assert_parity, run_gpu  # noqa: E402


def fuzz(pb, count, seed):
    rng = np.random.default_rng(seed)
    cs = gen.generate(pb, 0, count, p_mutate=0.2, p_bad=0.0)
    for x in range(count):
        kind = x % 6
        n = int(cs.n[x])
        if kind == 0:                                  # random split values
            q = int(rng.integers(0, cs.split.shape[1]))
            cs.split[x, q] = rng.integers(0, 16)
        elif kind == 1:                                # count off by a little
            cs.n[x] = max(0, n + int(rng.integers(-2, 3)))
        elif kind == 2:                                # ids out of range / padding inside
            p = int(rng.integers(0, max(1, n)))
            cs.fwd[x, p] = rng.choice([pb.n_max, pb.n_max + 7, 0xFFFF, int(rng.integers(0, pb.n_max))])
        elif kind == 3:                                # a duplicate in the backward order
            if n > 1:
                cs.bwd[x, 1] = cs.bwd[x, 0]
        elif kind == 4:                                # random bit rows
            cs.fb[x] = rng.integers(0, 2**32, cs.fb[x].shape, dtype=np.uint64).astype(np.uint32)
        else:                                          # garbage beyond n
            if n < pb.n_max:
                cs.bwd[x, n] = int(rng.integers(0, pb.n_max))
    return cs


@pytest.mark.parametrize("name,count,seed", [("toy", 600, 1), ("12B", 300, 2), ("T2V", 120, 3)])
def test_fuzzed_records_scorer(name, count, seed):
    pb = gen.make_problem(name)
    cs = fuzz(pb, count, seed)
    res, pk, win = run_gpu(pb, cs)
    assert_parity(pb, cs, res, pk, win)
    assert (res["status"] == oracle.ST_BAD).sum() > count // 3


@pytest.mark.parametrize("name,count,seed", [("toy", 300, 4), ("12B", 120, 5)])
def test_fuzzed_records_interleave_and_memopt(name, count, seed):
    from tests import test_gpu_interleave as TI
    from tests import test_gpu_memopt as TM
    pb = gen.make_problem(name)
    cs = fuzz(pb, count, seed)
    TI.check(pb, cs)
    TM.check(pb, cs)


def fuzz_orders(pb, ords, seed):
    """malformed per-rank orders: duplicates, a missing stage (0xFFFF inside), out-of-range ids,
    garbage beyond 2n, a backward before its forward (a cycle: DEADLOCK), swapped stages"""
    rng = np.random.default_rng(seed)
    o = ords.copy()
    for x in range(o.shape[0]):
        r = int(rng.integers(0, pb.P))
        row = o[x, r]
        m2 = int((row != 0xFFFF).sum())
        if m2 < 2:
            continue
        kind = x % 6
        a, b = (int(v) for v in rng.choice(m2, 2, replace=False))
        if kind == 0:
            row[b] = row[a]                                   # duplicate
        elif kind == 1:
            row[a] = 0xFFFF                                   # hole
        elif kind == 2:
            row[a] = (pb.n_max + int(rng.integers(0, 5))) | (int(row[a]) & 0x8000)   # id out of range
        elif kind == 3:
            if m2 < row.shape[0]:
                row[m2] = int(rng.integers(0, pb.n_max))      # garbage beyond 2n
        elif kind == 4:
            fpos = [t for t in range(m2) if not row[t] & 0x8000]
            s = int(row[fpos[-1]])
            bpos = [t for t in range(m2) if row[t] == (s | 0x8000)][0]
            row[fpos[-1]], row[bpos] = row[bpos], row[fpos[-1]]   # its backward first: a cycle
        else:
            row[a], row[b] = row[b], row[a]                   # any swap (valid or deadlocked)
    return o


@pytest.mark.parametrize("name,count,seed", [("toy", 300, 7), ("12B", 120, 8)])
def test_fuzzed_orders_eval_and_memopt(name, count, seed):
    """dip_eval_orders and dip_memopt on malformed per-rank orders: statuses, makespans, peaks (and
    the memopt re-timing) equal the oracle's explicit-order evaluation; nothing crashes"""
    pb = gen.make_problem(name)
    menu = strategy_menu(pb)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0.0, p_bad=0.0)
    rords, _ = oracle.interleave(pb, cs, threads=16)
    o = fuzz_orders(pb, rords, seed)
    m = dip.Model(pb, 0)
    m.set_strategies(menu, 10)
    ws = dip.Workspace(m)
    s = torch.cuda.current_stream()
    d_rec = torch.from_numpy(m.encode(cs)).cuda()
    d_ord = torch.from_numpy(o.view(np.int16)).cuda()
    d_res = torch.empty(count * 24, dtype=torch.uint8, device="cuda")
    d_pk = torch.empty((count, pb.P), dtype=torch.int32, device="cuda")
    dip.eval_orders(m, ws, d_rec, d_ord, count, d_res, d_pk, stream=s)
    torch.cuda.synchronize()
    res = dip.results_view(d_res.cpu().numpy()).copy()
    ref = oracle.evaluate(pb, cs, threads=16, orders=o)
    assert np.array_equal(res["status"], ref.status)
    assert np.array_equal(res["makespan_ns"], ref.makespan)
    assert np.array_equal(res["oom_mask"], ref.oom_mask)
    assert np.array_equal(d_pk.cpu().numpy().view(np.uint32).astype(np.uint64), ref.peaks)
    st = np.bincount(ref.status, minlength=4)
    assert st[oracle.ST_BAD] > 0 and st[oracle.ST_DEADLOCK] > 0
    d_sel = torch.empty(count * pb.P * 2 * pb.n_max, dtype=torch.uint8, device="cuda")
    dip.memopt(m, ws, d_rec, count, d_sel, d_res, d_pk, stream=s, d_orders=d_ord)
    torch.cuda.synchronize()
    res3 = dip.results_view(d_res.cpu().numpy())
    rsel, ref3 = oracle.memopt(pb, cs, menu, S=10, threads=16, orders=o)
    assert np.array_equal(res3["status"], ref3.status)
    assert np.array_equal(res3["makespan_ns"], ref3.makespan)
