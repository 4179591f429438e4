"""Pins of the CPU oracle against what the paper and mathematics fix (not against itself).

Every expected value here is either printed in PAPER.md, a closed form of a
textbook schedule, a brute-force count, or a hand-worked timeline (SURVEY.md
Appendix A, re-derived below where cheap). Citations: P:n = PAPER.md line n,
S:n = SPEC.md line n.
"""
from fractions import Fraction
import itertools

import numpy as np
import pytest

import oracle
from gen import Candidates, Module, Problem
from tests import helpers as H
from tests import refsim

OK, OOM, DL, BAD = oracle.ST_OK, oracle.ST_OOM, oracle.ST_DEADLOCK, oracle.ST_BAD


def ev(pb, cs):
    return oracle.evaluate(pb, cs, threads=1)


# ---------------------------------------------------------------- O1 / O2 -----
def test_chunking_spec_examples():
    # S:314-316 (examples of P:457-459): 16 chunks of 4; remainder to the earliest chunks; too many chunks
    assert oracle.chunk_layers(64, 16, 1) == [4] * 16
    assert oracle.chunk_layers(63, 4, 2) == [8, 8, 8, 8, 8, 8, 8, 7]
    assert oracle.chunk_layers(4, 4, 2) is None


def test_split_spec_examples_and_balance():
    # N=48,B=12 -> 4x12 ; N=10 -> [10] ; N=25 -> ceil(25/12)=3 parts [9,8,8]
    assert oracle.split_sizes(48, 4) == [12] * 4
    assert oracle.split_sizes(10, 1) == [10]
    assert oracle.split_sizes(25, 3) == [9, 8, 8]
    for N in range(1, 61):
        for M in range(1, min(N, 15) + 1):
            s = oracle.split_sizes(N, M)
            assert sum(s) == N and max(s) - min(s) <= 1 and s == sorted(s, reverse=True)


# ---------------------------------------------------------------- A.1 ---------
def test_h1_hand_timeline_1f1b_and_gpipe():
    # P=2, m=2, t_f=1, t_b=2 -> makespan 9, bubble 1/3, peaks [2a, a]
    a = 5
    pb = H.uniform_problem(2, 2, 1, 2, act=a)
    cs = H.candidates_from_orders(pb, [[1, 1], [1, 1]], [H.one_f_one_b(2, 2), H.gpipe(2, 2)])
    st, s, e = oracle.timeline(pb, cs, 0)
    assert st == OK
    # rank 0: F0 0-1, F1 1-2, B0 4-6, B1 7-9 ; rank 1: F0 1-2, B0 2-4, F1 4-5, B1 5-7
    assert s[0].tolist() == [0, 1, 4, 7] and e[0].tolist() == [1, 2, 6, 9]
    assert s[1].tolist() == [1, 2, 4, 5] and e[1].tolist() == [2, 4, 5, 7]
    r = ev(pb, cs)
    assert r.makespan.tolist() == [9, 9]
    assert r.bubble[0] == float(Fraction(1, 3)) and r.bubble[1] == float(Fraction(1, 3))
    assert r.peaks[0].tolist() == [2 * a, a] and r.peaks[1].tolist() == [2 * a, 2 * a]


# ---------------------------------------------------------------- A.2 ---------
def two_module_problem(P=2):
    vit = Module("vit", P, 1, 2, 1, 0, *H.table(1, {1: (1, 2, 3, 0)}))
    llm = Module("llm", P, 1, 1, 1, 1, *H.table(1, {1: (2, 4, 10, 0)}))
    off = np.array([0, 2, 3], np.uint32)        # 2 images (1 unit each), 1 text instance
    units = np.array([1, 1, 1], np.uint16)
    return Problem("h2", P, 1, [vit, llm], off, units, np.full(P, 1000, np.uint32))


def test_h2_two_module_join_timeline():
    # ViT split into 2 sub-microbatches, LLM one segment; order
    # F.V0 F.V1 F.L B.L B.V0 B.V1 on both ranks -> makespan 21, bubble 3/7, peak 16
    pb = two_module_problem()
    # ids: vit j=0 -> 0, j=1 -> 1, llm -> 2
    order = [("F", 0), ("F", 1), ("F", 2), ("B", 2), ("B", 0), ("B", 1)]
    cs = H.candidates_from_orders(pb, [[2, 1]], [[order, order]])
    st, s, e = oracle.timeline(pb, cs, 0)
    assert st == OK
    assert list(zip(s[0].tolist(), e[0].tolist())) == [(0, 1), (1, 2), (3, 5), (11, 15), (17, 19), (19, 21)]
    assert list(zip(s[1].tolist(), e[1].tolist())) == [(1, 2), (2, 3), (5, 7), (7, 11), (15, 17), (17, 19)]
    r = ev(pb, cs)
    assert int(r.makespan[0]) == 21 and r.bubble[0] == float(Fraction(3, 7))
    assert r.peaks[0].tolist() == [16, 16]


# ---------------------------------------------------------------- A.5 ---------
@pytest.mark.parametrize("tf,tb", [(1, 1), (1, 2), (2, 3)])
def test_1f1b_and_gpipe_closed_forms(tf, tb):
    # 1F1B / GPipe with uniform stages: makespan (m+P-1)(t_f+t_b), bubble (P-1)/(m+P-1)
    # (P=4, m=64 -> "≈ 4.48%" = 3/67), 1F1B peaks min(P-r, m)*a, GPipe peaks m*a.
    a = 3
    for P in range(1, 7):
        for m in range(1, 9):
            pb = H.uniform_problem(P, m, tf, tb, act=a)
            cs = H.candidates_from_orders(pb, [[1] * m] * 2, [H.one_f_one_b(P, m), H.gpipe(P, m)])
            r = ev(pb, cs)
            mk = (m + P - 1) * (tf + tb)
            assert r.makespan.tolist() == [mk, mk], (P, m)
            bub = float(Fraction(P - 1, m + P - 1))
            assert r.bubble.tolist() == [bub, bub]
            assert r.peaks[0].tolist() == [min(P - r_, m) * a for r_ in range(P)]
            assert r.peaks[1].tolist() == [m * a] * P
            assert r.status.tolist() == [OK, OK]


def test_spec_1f1b_bubble_example():
    # P=4, n=64, uniform -> bubble (P-1)/(n+P-1) "≈ 4.48%" (exactly 3/67 = 4.4776...%)
    pb = H.uniform_problem(4, 64, 1, 2)
    cs = H.candidates_from_orders(pb, [[1] * 64], [H.one_f_one_b(4, 64)])
    r = ev(pb, cs)
    assert round(r.bubble[0] * 100, 2) == 4.48 and r.bubble[0] == 3 / 67


# ---------------------------------------------------------------- A.4 ---------
@pytest.mark.parametrize("tf,tb", [(1, 2), (1, 1)])
def test_vpp_closed_form(tf, tb):
    # Megatron interleaved 1F1B with v chunks: makespan m*v*(t_f+t_b) + (P-1)(t_f+t_b),
    # bubble (P-1)/(v*m + P-1)
    for P in (2, 3, 4):
        for v in (1, 2, 3):
            for m in (P, 2 * P, 3 * P):
                pb = H.uniform_problem(P, m, tf, tb, K=v)
                cs = H.candidates_from_orders(pb, [[1] * m], [H.vpp(P, v, m)])
                r = ev(pb, cs)
                assert int(r.makespan[0]) == m * v * (tf + tb) + (P - 1) * (tf + tb), (P, v, m)
                assert r.bubble[0] == float(Fraction(P - 1, v * m + P - 1))


def test_vpp_example_peaks():
    # P=4, v=2, m=8, t_f=1, t_b=2 -> makespan 57, bubble 3/19, peaks [11, 9, 7, 5]*a
    pb = H.uniform_problem(4, 8, 1, 2, act=2, K=2)
    cs = H.candidates_from_orders(pb, [[1] * 8], [H.vpp(4, 2, 8)])
    r = ev(pb, cs)
    assert int(r.makespan[0]) == 57 and r.bubble[0] == 3 / 19
    assert r.peaks[0].tolist() == [22, 18, 14, 10]


# ---------------------------------------------------------------- A.3 ---------
def test_paper_s22_imbalance_example():
    # 64 ViT layers x 6.75 ms + 64 LM layers x 10.5 ms (fw+bw) over 16 stages; the
    # min-max partition gives stage latencies 63..73.5 ms ("16.7% variation"); 1F1B with 64
    # microbatches -> "22.8% additional pipeline bubbles".  One min-max partition (App. A.3):
    # 6 x 10 ViT | 4 ViT + 4 LM | 3 x 6 LM | 6 x 7 LM.  Layer unit = 0.25 ms of F (F:B = 1:2):
    # ViT layer = 9 units (2.25 + 4.5 ms), LM layer = 14 units (3.5 + 7.0 ms).
    chunks = [90] * 6 + [92] + [84] * 3 + [98] * 6
    fb_ms = [c * 0.25 * 3 for c in chunks]
    assert min(fb_ms) == 63.0 and max(fb_ms) == 73.5
    assert round((73.5 - 63.0) / 63.0 * 100, 1) == 16.7            # P:247 "16.7% variation"
    md = Module("mixed", sum(chunks), 1, 1, 1, 0, *H.table(1, {1: (250_000, 500_000, 1, 0)}),
                chunk_layers=np.array(chunks, np.uint32))
    m = 64
    pb = Problem("s22", 16, m, [md], np.arange(m + 1, dtype=np.uint32), np.ones(m, np.uint16),
                 np.full(16, 1 << 31, np.uint32))
    cs = H.candidates_from_orders(pb, [[1] * m], [H.one_f_one_b(16, m)])
    r = ev(pb, cs)
    assert int(r.makespan[0]) == 5_734_500_000
    assert r.bubble[0] == float(Fraction(879, 3823))
    assert abs(r.bubble[0] - 0.228) < 0.003                         # P:248 "22.8%"
    assert r.peaks[0].tolist() == [min(16 - k, m) * chunks[k] for k in range(16)]
    # the independent evaluator agrees exactly
    st, mk, pk, bub, busy = refsim.evaluate(pb, cs, 0)
    assert (st, mk, bub) == (OK, 5_734_500_000, r.bubble[0])


# ---------------------------------------------------------------- A.6 / A.7 ---
def _all_encodings(P, m):
    ids = list(range(m))
    bitsets = [b for b in itertools.product([0, 1], repeat=2 * m) if sum(b) == m]
    for fp in itertools.permutations(ids):
        for bp in itertools.permutations(ids):
            for rb in itertools.product(bitsets, repeat=P):
                yield fp, bp, rb


def _encode_all(pb, m, encs):
    encs = list(encs)
    cs = Candidates(pb, len(encs))
    cs.split[:] = 1
    cs.n[:] = m
    for c, (fp, bp, rb) in enumerate(encs):
        cs.fwd[c, :m] = fp
        cs.bwd[c, :m] = bp
        for r, bits in enumerate(rb):
            word = 0
            for t, bit in enumerate(bits):
                word |= bit << t
            cs.fb[c, r, 0] = word
    return cs


@pytest.mark.parametrize("P,m,tf,tb,total,valid,best", [
    (2, 2, 1, 2, 144, 8, 9), (3, 2, 1, 2, 864, 10, 12), (2, 3, 1, 2, 14400, 186, 12), (2, 3, 2, 3, 14400, 186, 20)])
def test_brute_force_whole_encoding_space(P, m, tf, tb, total, valid, best):
    # every fwd perm x bwd perm x per-rank bit string; the valid count does not
    # depend on latencies, and the optimum equals the 1F1B closed form (m+P-1)(t_f+t_b).
    pb = H.uniform_problem(P, m, tf, tb)
    cs = _encode_all(pb, m, _all_encodings(P, m))
    assert cs.count == total
    r = oracle.evaluate(pb, cs, threads=8)
    ok = r.status == OK
    assert int(ok.sum()) == valid
    assert int(r.makespan[ok].min()) == best == (m + P - 1) * (tf + tb)
    assert set(r.status.tolist()) <= {OK, DL}
    # deadlock verdicts agree with the independent evaluator (cycle found by DFS) on a sample
    for c in list(np.nonzero(ok)[0][:20]) + list(np.nonzero(~ok)[0][:60]):
        assert refsim.evaluate(pb, cs, int(c))[0] == int(r.status[c])


def test_deadlock_examples():
    # App. A.7 D1: rank 0 runs B0 before F0.  D2: P=2, m=2, rank 0 runs F0 B0 F1 B1 while rank 1
    # runs F0 F1 B0 B1 (warm-up increasing with rank): cycle B0@0 <- B0@1 <- F1@1 <- F1@0 <- B0@0.
    pb = H.uniform_problem(2, 2, 1, 2, act=1)
    d2 = [[("F", 0), ("B", 0), ("F", 1), ("B", 1)], [("F", 0), ("F", 1), ("B", 0), ("B", 1)]]
    pb1 = H.uniform_problem(2, 1, 1, 2, act=1)
    d1 = [[("B", 0), ("F", 0)], [("F", 0), ("B", 0)]]
    cs = H.candidates_from_orders(pb, [[1, 1]], [d2])
    cs1 = H.candidates_from_orders(pb1, [[1]], [d1])
    r, r1 = ev(pb, cs), ev(pb1, cs1)
    assert r.status[0] == DL and r1.status[0] == DL
    assert int(r.makespan[0]) == 2 ** 64 - 1 and r.bubble[0] == -1.0
    assert r.peaks[0].tolist() == [1, 2]           # peaks depend on order only (R-9)


# ---------------------------------------------------------------- A.9 ---------
def test_p2p_h1_timeline():
    # H1 with a transfer c=1 on every cross-rank edge -> makespan 11, bubble 5/11
    pb = H.uniform_problem(2, 2, 1, 2, p2p=1)
    cs = H.candidates_from_orders(pb, [[1, 1], [1, 1]], [H.one_f_one_b(2, 2), H.gpipe(2, 2)])
    st, s, e = oracle.timeline(pb, cs, 0)
    assert list(zip(s[0].tolist(), e[0].tolist())) == [(0, 1), (1, 2), (6, 8), (9, 11)]
    assert list(zip(s[1].tolist(), e[1].tolist())) == [(2, 3), (3, 5), (5, 6), (6, 8)]
    r = ev(pb, cs)
    assert r.makespan.tolist() == [11, 11] and r.bubble[0] == 5 / 11


def test_p2p_gpipe_closed_form_and_1f1b_counterexample():
    # GPipe: (m+P-1)(t_f+t_b) + 2(P-1)c for every c >= 0; 1F1B equals it only for m <= 2
    for tf, tb in [(1, 2), (2, 3)]:
        for P in range(1, 6):
            for m in range(1, 7):
                for c in (0, 1, 3, 8):
                    pb = H.uniform_problem(P, m, tf, tb, p2p=c)
                    cs = H.candidates_from_orders(pb, [[1] * m] * 2, [H.gpipe(P, m), H.one_f_one_b(P, m)])
                    r = ev(pb, cs)
                    closed = (m + P - 1) * (tf + tb) + 2 * (P - 1) * c
                    assert int(r.makespan[0]) == closed
                    if m <= 2:
                        assert int(r.makespan[1]) == closed
    pb = H.uniform_problem(2, 3, 1, 2, p2p=1)
    cs = H.candidates_from_orders(pb, [[1] * 3], [H.one_f_one_b(2, 3)])
    assert int(ev(pb, cs).makespan[0]) == 16          # not the GPipe formula's 14


# ---------------------------------------------------------------- status ------
def test_status_rules_and_sentinels():
    a = 4
    base = H.uniform_problem(2, 2, 1, 2, act=a, budget=[2 * a, a])       # 1F1B peaks [2a, a]
    good = H.candidates_from_orders(base, [[1, 1]], [H.one_f_one_b(2, 2)])
    r = ev(base, good)
    assert r.status[0] == OK                                             # equality fits (R-10)
    tight = H.uniform_problem(2, 2, 1, 2, act=a, budget=[2 * a - 1, a])
    r = ev(tight, good)
    assert r.status[0] == OOM and r.oom_mask[0] == 1 and int(r.makespan[0]) == 9   # OOM is timed
    # deadlock beats OOM (R-13)
    d2 = [[("F", 0), ("B", 0), ("F", 1), ("B", 1)], [("F", 0), ("F", 1), ("B", 0), ("B", 1)]]
    dl = H.candidates_from_orders(tight, [[1, 1]], [d2])
    assert ev(tight, dl).status[0] == DL
    # malformed encodings (R-11): each -> BAD, makespan UINT64_MAX, bubble -1, peaks 0, oom 0
    muts = []
    c = good.subset([0]); c.split[0, 0] = 2; muts.append(c)               # M > min(N, M_max)
    c = good.subset([0]); c.fwd[0, 1] = c.fwd[0, 0]; muts.append(c)       # duplicate id
    c = good.subset([0]); c.fb[0, 0, 0] ^= 1; muts.append(c)              # popcount != n
    c = good.subset([0]); c.n[0] = 1; muts.append(c)                      # n mismatch
    c = good.subset([0]); c.fb[0, 1, 0] |= 1 << 20; muts.append(c)        # bit beyond 2n
    for c in muts:
        r = ev(tight, c)
        assert r.status[0] == BAD and int(r.makespan[0]) == 2 ** 64 - 1
        assert r.bubble[0] == -1.0 and r.peaks[0].tolist() == [0, 0] and r.oom_mask[0] == 0


def test_pad_must_be_ffff():
    # ids beyond n must be the 0xFFFF pad (R-11)
    pb = two_module_problem()
    order = [("F", 0), ("F", 2), ("B", 2), ("B", 0)]
    c = H.candidates_from_orders(pb, [[1, 1]], [[order, order]])
    assert c.fwd[0].tolist() == [0, 2, 0xFFFF]
    assert ev(pb, c).status[0] == OK
    for bad in (1, 0, 0xFFFE):
        c2 = c.subset([0])
        c2.fwd[0, 2] = bad
        assert ev(pb, c2).status[0] == BAD


def test_empty_batch():
    # n = 0 (no instances at all): makespan 0, bubble 0.0, OK
    md = Module("m", 2, 1, 1, 1, 0, *H.table(1, {1: (1, 2, 1, 0)}))
    pb = Problem("e", 2, 2, [md], np.zeros(3, np.uint32), np.zeros(0, np.uint16), np.full(2, 9, np.uint32))
    cs = Candidates(pb, 1)
    r = ev(pb, cs)
    assert r.status[0] == OK and int(r.makespan[0]) == 0 and r.bubble[0] == 0.0


def test_argmin_ties_and_empty():
    # P:499-501 (best score), ties -> lowest index (R-15), no feasible -> -1
    ms = np.array([9, 7, 7, 5, 5], np.uint64)
    st = np.array([OK, OK, OK, OOM, DL], np.uint32)
    assert oracle.argmin(ms, st) == 1
    assert oracle.argmin(ms, np.full(5, OOM, np.uint32)) == -1
