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
