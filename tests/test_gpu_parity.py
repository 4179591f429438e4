"""GPU (sm_100a, through the C-ABI) vs the CPU oracle, element by element.

Makespans, statuses, OOM masks, per-rank peaks and the argmin must be bit-exact
(all integers); the bubble ratio within 1e-9 relative (BASELINE.json north_star)
-- it is in fact expected bit-identical (one IEEE division of exact integers).
"""
import copy

import numpy as np
import pytest

import gen
import oracle
from gen import Candidates, Module, Problem
from tests import helpers as H

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2504_14145_b200 as dip  # noqa: E402

BUBBLE_RTOL = 1e-9


def run_gpu(pb, cs, peaks=True):
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    recs = m.encode(cs)
    s = torch.cuda.current_stream()
    d_rec = torch.from_numpy(recs).cuda()
    d_res = torch.empty(max(1, cs.count) * 24, dtype=torch.uint8, device="cuda")
    d_pk = torch.empty((max(1, cs.count), pb.P), dtype=torch.int32, device="cuda") if peaks else None
    dip.eval_schedules(m, ws, d_rec, cs.count, d_res, d_pk, stream=s)
    win = dip.argmin(m, ws, cs.count, stream=s)
    torch.cuda.synchronize()
    res = dip.results_view(d_res.cpu().numpy())[:cs.count]
    pk = d_pk.cpu().numpy().view(np.uint32)[:cs.count] if peaks else None
    return res, pk, win


def assert_parity(pb, cs, res, pk, win):
    ref = oracle.evaluate(pb, cs, threads=16)
    assert np.array_equal(res["status"], ref.status), np.nonzero(res["status"] != ref.status)[0][:10]
    bad_mk = np.nonzero(res["makespan_ns"] != ref.makespan)[0]
    assert bad_mk.size == 0, (bad_mk[:10], res["makespan_ns"][bad_mk[:3]], ref.makespan[bad_mk[:3]])
    assert np.array_equal(res["oom_mask"], ref.oom_mask)
    b_gpu, b_ref = res["bubble"], ref.bubble
    assert np.all(np.abs(b_gpu - b_ref) <= BUBBLE_RTOL * np.abs(b_ref)), "bubble beyond 1e-9 relative"
    if pk is not None:
        assert np.array_equal(pk.astype(np.uint64), ref.peaks)
    best = oracle.argmin(ref.makespan, ref.status)
    assert win.found == (best >= 0)
    if best >= 0:
        assert win.global_index == best and win.makespan_ns == int(ref.makespan[best])
    return int(np.sum(b_gpu.view(np.uint64) == b_ref.view(np.uint64)))


@pytest.mark.parametrize("name,count", [("toy", 256), ("12B", 4096), ("37B", 2048), ("T2V", 1024), ("94B", 512)])
def test_parity_configs(name, count):
    pb = gen.make_problem(name)
    if name == "toy":
        cs = gen.generate(pb, 0, count, mode=1)
    else:
        cs = gen.generate(pb, 0, count, p_mutate=0.15, p_bad=0.03)
    res, pk, win = run_gpu(pb, cs)
    exact = assert_parity(pb, cs, res, pk, win)
    assert exact == count     # bubble bit-identical too
    st = np.bincount(res["status"], minlength=4)
    if name != "toy":
        assert st[0] > 0 and st[2] > 0 and st[3] > 0      # OK, DEADLOCK and BAD all exercised


def test_parity_12B_full_size():
    # BASELINE.json configs[1]: 64K candidates of the 12B VLM, every one checked
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 65536)
    res, pk, win = run_gpu(pb, cs, peaks=True)
    assert_parity(pb, cs, res, pk, win)


@pytest.mark.parametrize("name", ["37B", "T2V", "94B"])
def test_parity_full_population(name):
    """BASELINE.json configs[2..4] at their full per-GPU size (1,048,576 candidates -- for 94B the
    per-GPU shard of the 8M batch, the bench's launch), EVERY candidate against the oracle on all host
    cores: status, makespan, OOM mask, per-rank peaks, bubble and the argmin"""
    import os
    pb = gen.make_problem(name)
    N = 1 << 20
    cs = gen.generate(pb, 0, N, threads=os.cpu_count() or 1)
    res, pk, win = run_gpu(pb, cs, peaks=True)
    ref = oracle.evaluate(pb, cs, threads=os.cpu_count() or 1)
    assert np.array_equal(res["status"], ref.status), np.nonzero(res["status"] != ref.status)[0][:10]
    assert np.array_equal(res["makespan_ns"], ref.makespan), np.nonzero(res["makespan_ns"] != ref.makespan)[0][:10]
    assert np.array_equal(res["oom_mask"], ref.oom_mask)
    assert np.array_equal(res["bubble"].view(np.uint64), ref.bubble.view(np.uint64))
    assert np.array_equal(pk.astype(np.uint64), ref.peaks)
    best = oracle.argmin(ref.makespan, ref.status)
    assert win.found == (best >= 0) and win.global_index == best and win.makespan_ns == int(ref.makespan[best])
    st = np.bincount(res["status"], minlength=4)
    assert st.min() > 0                       # OK, OOM, DEADLOCK and BAD_ENCODING all present
    print(f"RESULT {name} full population: {N} candidates identical, status histogram {st.tolist()}")


def _spill_problem():
    return H.uniform_problem(4, 32, 3, 5, act=1, p2p=2)


def test_channel_spill_long_leads():
    # rank 0 runs GPipe (all forwards first) while ranks 1..3 run 1F1B: rank 0 leads rank 1 by up
    # to 29 forwards and rank 1 leads rank 0 by up to 29 backwards -> both channels spill (RING_D = 8)
    P, m = 4, 32
    pb = _spill_problem()
    one = H.one_f_one_b(P, m)
    gp = H.gpipe(P, m)
    mixes = [[gp[0]] + one[1:], [gp[0], gp[1]] + one[2:], gp[:3] + one[3:], one, gp]
    cs = H.candidates_from_orders(pb, [[1] * m] * len(mixes), mixes)
    res, pk, win = run_gpu(pb, cs)
    assert_parity(pb, cs, res, pk, win)
    assert (res["status"] == 0).all()


def test_single_rank_and_empty_batch():
    pb = gen.make_problem("toy")
    pb1 = copy.deepcopy(pb)
    pb1.P = 1
    pb1.budget_kib = pb.budget_kib[:1].copy()
    cs = gen.generate(pb1, 0, 256, mode=1)
    res, pk, win = run_gpu(pb1, cs)
    assert_parity(pb1, cs, res, pk, win)
    md = Module("m", 2, 1, 1, 1, 0, *H.table(1, {1: (1, 2, 1, 0)}))
    pbe = Problem("e", 2, 2, [md], np.zeros(3, np.uint32), np.zeros(0, np.uint16), np.full(2, 9, np.uint32))
    cse = Candidates(pbe, 3)
    res, pk, win = run_gpu(pbe, cse)
    assert_parity(pbe, cse, res, pk, win)
    assert (res["makespan_ns"] == 0).all() and win.found and win.global_index == 0


def test_paper_pins_on_gpu():
    # the §2.2 example and the VPP / p2p closed forms, straight through the kernel
    chunks = [90] * 6 + [92] + [84] * 3 + [98] * 6
    md = Module("mixed", sum(chunks), 1, 1, 1, 0, *H.table(1, {1: (250_000, 500_000, 1, 0)}),
                chunk_layers=np.array(chunks, np.uint32))
    pb = Problem("s22", 16, 64, [md], np.arange(65, dtype=np.uint32), np.ones(64, np.uint16),
                 np.full(16, 1 << 31, np.uint32))
    cs = H.candidates_from_orders(pb, [[1] * 64], [H.one_f_one_b(16, 64)])
    res, pk, win = run_gpu(pb, cs)
    assert int(res["makespan_ns"][0]) == 5_734_500_000 and res["bubble"][0] == 879 / 3823
    for P, v, m in [(4, 2, 8), (3, 3, 6), (2, 1, 4)]:
        pbv = H.uniform_problem(P, m, 1, 2, K=v, p2p=0)
        csv = H.candidates_from_orders(pbv, [[1] * m], [H.vpp(P, v, m)])
        res, pk, win = run_gpu(pbv, csv)
        assert int(res["makespan_ns"][0]) == m * v * 3 + (P - 1) * 3
    pbp = H.uniform_problem(3, 5, 1, 2, p2p=4)
    csp = H.candidates_from_orders(pbp, [[1] * 5], [H.gpipe(3, 5)])
    res, pk, win = run_gpu(pbp, csp)
    assert int(res["makespan_ns"][0]) == (5 + 2) * 3 + 2 * 2 * 4


def test_argmin_exact_fallback_when_key_could_overflow():
    # latencies near 2^46 ns make the packed (makespan << idx_bits | index) key unsafe for 32K
    # candidates, so the library takes the exact two-pass scan; ties -> lowest index (R-15)
    md = Module("big", 1, 1, 1, 1, 0, *H.table(1, {1: (2 ** 31, 2 ** 32 - 1, 1, 0)}),
                chunk_layers=np.array([16384], np.uint32))
    pb = Problem("big", 1, 8, [md], np.arange(9, dtype=np.uint32), np.ones(8, np.uint16),
                 np.full(1, 1 << 30, np.uint32))
    m = dip.Model(pb, 0)
    assert m.info["makespan_bound"] >= 2 ** 49
    N = 1 << 15
    orders = [H.one_f_one_b(1, 8), H.gpipe(1, 8)]
    cs = H.candidates_from_orders(pb, [[1] * 8] * N, [orders[x % 2] for x in range(N)])
    cs.fb[5, 0, 0] ^= 1          # one bad encoding
    res, pk, win = run_gpu(pb, cs)
    assert_parity(pb, cs, res, pk, win)
    assert win.found and win.global_index == 0


def test_host_end_to_end_path():
    pb = gen.make_problem("37B")
    cs = gen.generate(pb, 0, 5000)
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m, host_chunk=1024)
    recs = torch.from_numpy(m.encode(cs)).pin_memory()
    h_res = np.zeros(cs.count * 24, np.uint8)
    win = dip.eval_host(m, ws, recs, cs.count, h_results=h_res, stream=torch.cuda.current_stream())
    ref = oracle.evaluate(pb, cs, threads=16)
    r = dip.results_view(h_res)
    assert np.array_equal(r["makespan_ns"], ref.makespan) and np.array_equal(r["status"], ref.status)
    best = oracle.argmin(ref.makespan, ref.status)
    assert win.found and win.global_index == best


def test_maximum_shapes():
    # the record format's extremes: P = 32 ranks and m = 255 microbatches (the u8 microbatch field),
    # K = 4 chunks -> n = 1020 segments, 65,280 stage nodes per candidate: chunk-major forward order,
    # reversed backward order; per-rank warm-ups n - 2r (then 1F1B), all-forward-first (GPipe), and
    # one adjacent F/B swap -- bit-exact against the oracle
    P, m, K = 32, 255, 4
    n = m * K
    pb = H.uniform_problem(P, m, 3, 5, act=2, p2p=1, K=K, budget=[4000] * P)
    fseq = [b * K + k for k in range(K) for b in range(m)]
    bseq = [b * K + k for k in reversed(range(K)) for b in range(m)]

    def ranks(warm):
        out = []
        for r in range(P):
            w = warm(r)
            seq = [("F", s) for s in fseq[:w]]
            f, b = w, 0
            while b < n:
                seq.append(("B", bseq[b]))
                b += 1
                if f < n:
                    seq.append(("F", fseq[f]))
                    f += 1
            out.append(seq)
        return out

    orders = [ranks(lambda r: n - 2 * r), ranks(lambda r: n)]
    cs = H.candidates_from_orders(pb, [[1] * m] * 2, orders)
    cs2 = cs.subset([0, 1, 0])
    fb = cs2.fb[2, 7].copy()
    bits = [(int(fb[t >> 5]) >> (t & 31)) & 1 for t in range(2 * n)]
    t = next(t for t in range(1000, 2 * n - 1) if bits[t] != bits[t + 1])
    bits[t], bits[t + 1] = bits[t + 1], bits[t]
    cs2.fb[2, 7] = 0
    for i, bit in enumerate(bits):
        if bit:
            cs2.fb[2, 7, i >> 5] |= np.uint32(1 << (i & 31))
    res, pk, win = run_gpu(pb, cs2)
    assert_parity(pb, cs2, res, pk, win)
    assert res["status"][0] in (oracle.ST_OK, oracle.ST_OOM) and res["status"][1] in (oracle.ST_OK, oracle.ST_OOM)


def test_working_set_too_large_is_rejected():
    # n_max = 255 * 64 segments: the per-candidate shared-memory working set cannot fit -> DIP_ERANGE
    pb = H.uniform_problem(2, 255, 1, 2, K=64)
    with pytest.raises(dip.DipError) as e:
        dip.Model(pb, 0)
    assert e.value.code == 4
