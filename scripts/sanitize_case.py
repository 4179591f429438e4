"""Small scoring cases for compute-sanitizer (memcheck / racecheck / synccheck): every config,
the channel-spill case and the single-rank case, each checked against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2504_14145_b200 as dip  # noqa: E402
from tests import helpers as H  # noqa: E402


def run(pb, cs):
    m = dip.Model(pb, 0)
    ws = dip.Workspace(m)
    d_rec = torch.from_numpy(m.encode(cs)).cuda()
    d_res = torch.empty(cs.count * 24, dtype=torch.uint8, device="cuda")
    d_pk = torch.empty((cs.count, pb.P), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    dip.eval_schedules(m, ws, d_rec, cs.count, d_res, d_pk, stream=s)
    win = dip.argmin(m, ws, cs.count, stream=s)
    res = dip.results_view(d_res.cpu().numpy())
    ref = oracle.evaluate(pb, cs, threads=8)
    assert np.array_equal(res["makespan_ns"], ref.makespan) and np.array_equal(res["status"], ref.status)
    assert np.array_equal(d_pk.cpu().numpy().view(np.uint32).astype(np.uint64), ref.peaks)
    best = oracle.argmin(ref.makespan, ref.status)
    assert win.found == (best >= 0) and (best < 0 or win.global_index == best)


for name, cnt in [("toy", 256), ("12B", 256), ("37B", 96), ("T2V", 64), ("94B", 32)]:
    pb = gen.make_problem(name)
    cs = gen.generate(pb, 0, cnt, mode=1 if name == "toy" else 0, p_mutate=0.2, p_bad=0.05)
    run(pb, cs)
    print("ok", name, flush=True)
P, m = 4, 32
pb = H.uniform_problem(P, m, 3, 5, act=1, p2p=2)
one, gp = H.one_f_one_b(P, m), H.gpipe(P, m)
cs = H.candidates_from_orders(pb, [[1] * m] * 3, [[gp[0]] + one[1:], gp[:3] + one[3:], gp])
run(pb, cs)
print("ok spill", flush=True)
print("SANITIZE CASES PASSED")
