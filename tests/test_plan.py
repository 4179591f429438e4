"""f4 (§6.3): schedule -> per-rank action lists, checked on the
host with timelines from the CPU oracle: the hand-compiled 2-rank example, pairing
completeness and round-trip fidelity of the discrete-event execution, batching, and
rejection of broken plans."""
import numpy as np
import pytest

import gen
import oracle
from tests import helpers as H

ACT = ["fw_stage", "bw_stage", "isend", "irecv", "wait_isend", "wait_irecv"]


@pytest.fixture(scope="module")
def dip():
    from paper_2504_14145_b200 import build
    build.build()
    import paper_2504_14145_b200 as d
    return d


def oracle_rows(pb, cs, x):
    """oracle timeline padded to the [P, 2*n_max] rows the library uses"""
    st, s, e = oracle.timeline(pb, cs, x)
    S = np.zeros((pb.P, 2 * pb.n_max), np.uint64)
    E = np.zeros_like(S)
    if s is not None:
        S[:, : s.shape[1]] = s
        E[:, : e.shape[1]] = e
    return st, S, E


def compile_one(dip, pb, cs, x):
    m = dip.Model(pb, -1)
    rec = m.encode(cs.subset([x]))
    st, S, E = oracle_rows(pb, cs, x)
    acts, off, nmsg = dip.compile_plan(m, rec, S, E)
    return m, rec, st, S, acts, off, nmsg


def test_two_rank_hand_compilation(dip):
    # S:588 "2-rank, 1-microbatch, 1-segment forward -> rank0: [fw_stage, isend, wait_isend];
    # rank1: [irecv, wait_irecv, fw_stage]" -- here with the backward pass as well
    pb = H.uniform_problem(2, 1, 1, 2, p2p=1)
    cs = H.candidates_from_orders(pb, [[1]], [H.one_f_one_b(2, 1)])
    m, rec, st, S, acts, off, nmsg = compile_one(dip, pb, cs, 0)
    r0 = [ACT[a[0]] for a in acts[off[0]:off[1]]]
    r1 = [ACT[a[0]] for a in acts[off[1]:off[2]]]
    assert r0 == ["fw_stage", "isend", "irecv", "wait_isend", "wait_irecv", "bw_stage"]
    assert r1 == ["irecv", "wait_irecv", "fw_stage", "bw_stage", "isend", "wait_isend"]
    assert nmsg == 2


def _edges(pb, cs, x):
    """independent count of cross-rank dependency edges (R-4, R-5)"""
    P, nm = pb.P, pb.nmod
    if P == 1:
        return 0
    split = cs.split[x].reshape(pb.m, nm).astype(int)
    n = int(cs.n[x])
    dec = pb.seg_decode()
    tot = 0
    for s in cs.fwd[x][:n]:
        b, i, j, k = dec[int(s)]
        tot += P - 1                                           # F(s, r-1) -> F(s, r)
        tot += 1 if k > 0 else sum(int(split[b, p]) for p in range(nm) if (pb.modules[i].producer_mask >> p) & 1)
    for s in cs.bwd[x][:n]:
        b, i, j, k = dec[int(s)]
        tot += P - 1
        if k < pb.modules[i].K - 1:
            tot += 1
        else:
            tot += sum(int(split[b, c]) for c in range(nm) if (pb.modules[c].producer_mask >> i) & 1)
    return tot


@pytest.mark.parametrize("name,count", [("toy", 24), ("12B", 8), ("T2V", 4), ("37B", 3)])
def test_round_trip_fidelity_and_pairing(dip, name, count):
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, count, mode=1 if name == "toy" else 0, p_mutate=0, p_bad=0)
    for x in range(count):
        m, rec, st, S, acts, off, nmsg = compile_one(dip, pb, cs, x)
        if st not in (oracle.ST_OK, oracle.ST_OOM):
            continue
        kinds = acts[:, 0]
        assert (kinds == 2).sum() == (kinds == 3).sum() == (kinds == 4).sum() == (kinds == 5).sum() == nmsg
        assert nmsg == _edges(pb, cs, x)
        assert ((kinds == 0) | (kinds == 1)).sum() == pb.P * 2 * int(cs.n[x])
        ok, D = dip.validate_plan(m, rec, acts, off)
        assert ok
        assert np.array_equal(D, S)                 # every stage starts at its simulated time


def test_single_rank_plan_has_no_communication(dip):
    pb = gen.make_problem("toy")
    import copy
    pb1 = copy.deepcopy(pb)
    pb1.P = 1
    pb1.budget_kib = pb.budget_kib[:1].copy()
    cs = gen.generate(pb1, 0, 2, mode=1)
    m, rec, st, S, acts, off, nmsg = compile_one(dip, pb1, cs, 0)
    assert nmsg == 0 and set(acts[:, 0].tolist()) <= {0, 1}


def test_batching_groups_consecutive_p2p(dip):
    pb = gen.make_problem("12B")
    cs = gen.generate(pb, 0, 1, p_mutate=0, p_bad=0)
    m, rec, st, S, acts, off, nmsg = compile_one(dip, pb, cs, 0)
    for r in range(pb.P):
        a = acts[off[r]:off[r + 1]]
        prev_p2p, prev_batch = False, 0
        for kind, peer, tag, batch, slot in a:
            p2p = kind in (2, 3)
            if p2p:
                assert batch > 0 and (batch == prev_batch if prev_p2p else batch != prev_batch)
                prev_batch = batch
            else:
                assert batch == 0
            prev_p2p = p2p


def test_broken_plans_are_rejected(dip):
    pb = H.uniform_problem(2, 2, 1, 2, p2p=1)
    cs = H.candidates_from_orders(pb, [[1, 1]], [H.one_f_one_b(2, 2)])
    m, rec, st, S, acts, off, nmsg = compile_one(dip, pb, cs, 0)
    assert dip.validate_plan(m, rec, acts, off)[0]
    bad = acts.copy()
    i = int(np.nonzero(bad[:, 0] == 3)[0][0])
    bad[i, 2] = (bad[i, 2] + 1) % nmsg                      # an irecv with another message's tag
    assert not dip.validate_plan(m, rec, bad, off)[0]
    # rank 1 waits for its receive before rank 0 ever sends: move rank 0's first isend to its end
    r0 = acts[off[0]:off[1]].copy()
    k = int(np.nonzero(r0[:, 0] == 2)[0][0])
    moved = np.concatenate([r0[:k], r0[k + 1:], r0[k:k + 1]])
    # and make rank 0 wait for rank 1's backward first: a cycle through the waits
    dead = np.concatenate([moved, acts[off[1]:]])
    assert not dip.validate_plan(m, rec, dead, off)[0]


def test_malformed_records_and_orders_are_rejected(dip):
    """a record whose forward sequence repeats a segment, or per-rank orders with a duplicated /
    missing stage, is DIP_EINVAL for compile and validate -- not a crash (an id that never gets a
    slot used to index the post lists out of range)"""
    from paper_2504_14145_b200.dip import DipError
    pb = H.uniform_problem(4, 4, 1, 2, K=2, p2p=1)
    cs = H.candidates_from_orders(pb, [[1] * 4], [H.vpp(4, 2, 4)])
    m = dip.Model(pb, -1)
    st, S, E = oracle_rows(pb, cs, 0)
    good = m.encode(cs)
    acts, off, nmsg = dip.compile_plan(m, good, S, E)
    bad = cs.subset([0])
    bad.fwd[0, 1] = bad.fwd[0, 0]
    with pytest.raises(DipError) as e:
        dip.compile_plan(m, m.encode(bad), S, E)
    assert e.value.code == 1
    with pytest.raises(DipError):
        dip.validate_plan(m, m.encode(bad), acts, off)
    ords = H.orders_array(pb, H.vpp(4, 2, 4))
    acts2, off2, _ = dip.compile_plan(m, good, S, E, orders=ords)      # the same schedule as orders
    assert np.array_equal(acts2, acts) and np.array_equal(off2, off)
    for mut in ("dup", "missing"):
        o2 = ords.copy()
        if mut == "dup":
            o2[2, 3] = o2[2, 2] if (o2[2, 2] & 0x8000) == (o2[2, 3] & 0x8000) else o2[2, 1]
        else:
            o2[1, 0] = 0xFFFF
        with pytest.raises(DipError):
            dip.compile_plan(m, good, S, E, orders=o2)


def test_validator_rejects_out_of_range_actions(dip):
    """caller-supplied plans: a stage slot beyond 2n, a stage of the wrong direction, or a wait on an
    unknown tag make the plan invalid (ok = 0) instead of indexing out of range"""
    pb = H.uniform_problem(2, 2, 1, 2, p2p=1)
    cs = H.candidates_from_orders(pb, [[1, 1]], [H.one_f_one_b(2, 2)])
    m, rec, st, S, acts, off, nmsg = compile_one(dip, pb, cs, 0)
    ok, _ = dip.validate_plan(m, rec, acts, off)
    assert ok
    for field, kind, value in [(4, 0, 99), (0, 0, 1), (2, 4, 1000), (2, 5, 1000)]:
        a = acts.copy()
        x = int(np.nonzero(a[:, 0] == kind)[0][0])
        if field == 0:
            a[x, 0] = value             # fw_stage -> bw_stage at a forward slot
        else:
            a[x, field] = value
        ok, _ = dip.validate_plan(m, rec, a, off)
        assert not ok, (field, kind, value)
