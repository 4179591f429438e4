"""The C-ABI library without a GPU: it loads, exports every symbol include/dip.h declares,
validates problems at load time, and packs candidates into the documented record layout."""
import copy
import os
import re

import numpy as np
import pytest

import gen
from tests import helpers as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dip():
    from paper_2504_14145_b200 import build
    build.build()
    import paper_2504_14145_b200 as d
    return d


def test_library_exports_every_declared_symbol(dip):
    hdr = open(os.path.join(ROOT, "include", "dip.h")).read()
    names = set(re.findall(r"^\s*(?:dip_status|const char \*|uint64_t)\s*(dip_\w+)\s*\(", hdr, re.M))
    assert {"dip_load_cost_model", "dip_encode_candidates", "dip_eval_schedules", "dip_argmin"} <= names
    L = dip.lib()
    for n in sorted(names):
        assert hasattr(L, n), n


def _hostmodel(dip, pb):
    return dip.Model(pb, device=-1)


@pytest.mark.parametrize("name", gen.CONFIG_NAMES)
def test_host_model_shapes(dip, name):
    pb = gen.make_problem(name)
    m = _hostmodel(dip, pb)
    assert m.n_max == pb.n_max and m.fbw == pb.fbw and m.stride % 16 == 0
    assert m.info["group_lanes"] >= pb.P and 32 % m.info["group_lanes"] == 0


def test_load_time_validation(dip):
    pb = H.uniform_problem(4, 4, 1, 2)
    bad = copy.deepcopy(pb)
    bad.P = 33
    bad.budget_kib = np.ones(33, np.uint32)
    with pytest.raises(dip.DipError, match="EINVAL"):
        _hostmodel(dip, bad)
    bad = copy.deepcopy(pb)
    bad.modules[0].L = 3                       # P*K > L (S:316 TooManyChunks)
    with pytest.raises(dip.DipError, match="EINVAL"):
        _hostmodel(dip, bad)
    bad = copy.deepcopy(pb)
    bad.inst_units = np.full(4, 2, np.uint16)  # W = 2 > w_max = 1
    with pytest.raises(dip.DipError, match="ERANGE"):
        _hostmodel(dip, bad)
    pb2 = gen.make_problem("toy")
    bad = copy.deepcopy(pb2)
    bad.modules[0].producer_mask = 0b10        # a module fed by a later one
    with pytest.raises(dip.DipError, match="EINVAL"):
        _hostmodel(dip, bad)


def _decode(m, pb, rec):
    """Test-side reader of the record layout documented in include/dip.h."""
    n_pad = (pb.n_max + 7) // 8 * 8
    nsplit = sum(1 for md in pb.modules if md.max_split > 1)
    off_fwd = (4 + (pb.m * nsplit + 1) // 2 + 15) // 16 * 16
    off_bwd = off_fwd + 2 * n_pad
    off_fb = (off_bwd + 2 * n_pad + 15) // 16 * 16
    n, flags = np.frombuffer(rec[:4].tobytes(), np.uint16)
    nib = rec[4:off_fwd]
    fwd = np.frombuffer(rec[off_fwd:off_bwd].tobytes(), np.uint16)
    bwd = np.frombuffer(rec[off_bwd:off_bwd + 2 * n_pad].tobytes(), np.uint16)
    fb = np.frombuffer(rec[off_fb:off_fb + 4 * pb.fbw * pb.P].tobytes(), np.uint32).reshape(pb.fbw, pb.P).T
    split = []
    for b in range(pb.m):
        s = 0
        for i, md in enumerate(pb.modules):
            if md.max_split > 1:
                k = b * nsplit + s
                split.append((int(nib[k // 2]) >> (4 * (k % 2))) & 15)
                s += 1
    return int(n), int(flags), split, fwd, bwd, fb


@pytest.mark.parametrize("name", ["toy", "12B", "T2V", "94B"])
def test_encode_layout_roundtrip(dip, name):
    pb = gen.make_problem(name)
    m = _hostmodel(dip, pb)
    cs = gen.generate(pb, 0, 32, mode=1 if name == "toy" else 0, p_bad=0.0)
    recs = m.encode(cs).reshape(32, m.stride)
    for x in range(32):
        n, flags, split, fwd, bwd, fb = _decode(m, pb, recs[x])
        assert n == cs.n[x] and flags == 0
        sp = cs.split[x].reshape(pb.m, pb.nmod)
        assert split == [int(sp[b, i]) for b in range(pb.m) for i, md in enumerate(pb.modules) if md.max_split > 1]
        assert np.array_equal(fwd[:pb.n_max], cs.fwd[x]) and (fwd[pb.n_max:] == 0xFFFF).all()
        assert np.array_equal(bwd[:pb.n_max], cs.bwd[x]) and (bwd[pb.n_max:] == 0xFFFF).all()
        assert np.array_equal(fb, cs.fb[x])


def test_encode_flags_unrepresentable(dip):
    pb = gen.make_problem("12B")
    m = _hostmodel(dip, pb)
    cs = gen.generate(pb, 0, 4, p_bad=0.0)
    c = cs.subset([0, 1, 2, 3])
    c.n[0] = pb.n_max + 1                      # n > n_max
    c.split[1, 0] = 16                         # does not fit a nibble
    c.split[2, 1] = 2                          # module with M_max = 1: only the implied value is valid
    recs = m.encode(c).reshape(4, m.stride)
    assert [int(np.frombuffer(recs[x, 2:4].tobytes(), np.uint16)[0]) for x in range(4)] == [1, 1, 1, 0]
