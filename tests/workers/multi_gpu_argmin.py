"""torchrun worker for tests/test_gpu_multi.py: every rank scores its contiguous shard on its own
B200 through libdip, dip_argmin reduces the packed key with one ncclAllReduce over NVLink, and
rank 0 checks the winner against the CPU oracle over the whole batch."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import gen  # noqa: E402
import paper_2504_14145_b200 as dip  # noqa: E402
from tests import helpers as H  # noqa: E402


def score(pb, cs, model, ws, rank, world, comm, stride):
    d_rec = torch.from_numpy(model.encode(cs)).cuda()
    d_res = torch.empty(cs.count * 24, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    dip.eval_schedules(model, ws, d_rec, cs.count, d_res, None, stream=s)
    return dip.argmin(model, ws, cs.count, stride, rank, world, comm, stream=s)


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [dip.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = dip.Comm(obj[0], rank, world, local)
    out = {}
    # 1) packed single-allreduce path, 12B config
    pb = gen.make_problem("12B")
    S = 4096
    cs = gen.generate(pb, rank * S, S)
    m = dip.Model(pb, local)
    ws = dip.Workspace(m)
    win = score(pb, cs, m, ws, rank, world, comm, S)
    out["packed"] = [win.found, win.rank, win.global_index, win.makespan_ns]
    # 2) exact two-allreduce fallback (a makespan bound too large for the packed key)
    md = gen.Module("big", 1, 1, 1, 1, 0, *H.table(1, {1: (2 ** 31, 2 ** 32 - 1, 1, 0)}),
                    chunk_layers=np.array([16384], np.uint32))
    pbb = gen.Problem("big", 1, 8, [md], np.arange(9, dtype=np.uint32), np.ones(8, np.uint16),
                      np.full(1, 1 << 30, np.uint32))
    N = 1 << 15
    orders = [H.one_f_one_b(1, 8), H.gpipe(1, 8)]
    csb = H.candidates_from_orders(pbb, [[1] * 8] * N, [orders[(x + rank) % 2] for x in range(N)])
    mb = dip.Model(pbb, local)
    wsb = dip.Workspace(mb)
    winb = score(pbb, csb, mb, wsb, rank, world, comm, N)
    out["fallback"] = [winb.found, winb.rank, winb.global_index, winb.makespan_ns]
    if rank == 0:
        import oracle
        full = gen.generate(pb, 0, S * world)
        r = oracle.evaluate(pb, full, threads=os.cpu_count() or 1)
        best = oracle.argmin(r.makespan, r.status)
        out["oracle_packed"] = [best, int(r.makespan[best])]
        rb = oracle.evaluate(pbb, csb, threads=os.cpu_count() or 1)   # rank 0's shard holds the earliest tie
        bb = oracle.argmin(rb.makespan, rb.status)
        out["oracle_fallback"] = [bb, int(rb.makespan[bb])]
        ok = (win.found and win.global_index == best and win.makespan_ns == int(r.makespan[best]) and
              winb.found and winb.global_index == bb and winb.makespan_ns == int(rb.makespan[bb]))
        out["ok"] = bool(ok)
        print("RESULT " + json.dumps(out), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
