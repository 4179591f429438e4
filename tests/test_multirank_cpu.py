"""World-size-2 gloo test of the N>1 host logic on CPU: contiguous rank-major shards generated
independently per rank, the packed (makespan, rank, index) key of dip_argmin (libdip host
helpers), a MIN all-reduce, and the tie rule (lowest global index wins, R-15).

The per-rank local scores come from the CPU oracle here (no GPU); on a B200 the same key is
built by the kernel epilogue and reduced by ncclAllReduce (tests/test_gpu_multi.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SHARD = 192


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tie, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        import oracle
        import paper_2504_14145_b200 as dip
        pb = gen.make_problem("12B")
        first = 0 if tie else rank * SHARD
        cs = gen.generate(pb, first, SHARD, threads=2)
        full = gen.generate(pb, 0, SHARD * world, threads=2)
        if not tie:   # the generator is indexable: a shard equals the slice of the whole batch
            sl = slice(rank * SHARD, (rank + 1) * SHARD)
            assert np.array_equal(cs.fb, full.fb[sl]) and np.array_equal(cs.fwd, full.fwd[sl])
        r = oracle.evaluate(pb, cs, threads=2)
        best = oracle.argmin(r.makespan, r.status)
        key = dip.pack_key(int(r.makespan[best]), rank, best, SHARD, world) if best >= 0 else (1 << 64) - 1
        t = torch.tensor([key - (1 << 63)], dtype=torch.int64)   # order-preserving shift into int64
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        win = dip.unpack_key(int(t.item()) + (1 << 63), SHARD, world)
        if tie:
            exp_idx = best                                # identical shards: rank 0 wins every tie
            exp_mk = int(r.makespan[best])
        else:
            rf = oracle.evaluate(pb, full, threads=2)
            exp_idx = oracle.argmin(rf.makespan, rf.status)
            exp_mk = int(rf.makespan[exp_idx])
        out_q.put((rank, win.found, win.global_index, win.makespan_ns, exp_idx, exp_mk))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tie", [False, True])
def test_two_rank_argmin_over_gloo(tie):
    from paper_2504_14145_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tie, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, found, gidx, mk, exp_idx, exp_mk in res:
        assert found and gidx == exp_idx and mk == exp_mk, (rank, gidx, exp_idx)
