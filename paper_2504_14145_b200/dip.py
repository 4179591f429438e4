"""Thin ctypes binding of libdip.so (include/dip.h). Argument marshalling only:
every step of the scoring path runs in the library's sm_100a kernels.

PyTorch is used by callers for device memory, streams and process groups; this
module takes raw pointers (tensor.data_ptr()) or numpy arrays, and fails loudly
if the compiled library is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdip.so")

DIP_OK = 0
CAND_OK, CAND_OOM, CAND_DEADLOCK, CAND_BAD = 0, 1, 2, 3

RESULT_DTYPE = np.dtype([("makespan_ns", "<u8"), ("status", "<u4"), ("oom_mask", "<u4"), ("bubble", "<f8")])
assert RESULT_DTYPE.itemsize == 24

_u8p = ctypes.POINTER(ctypes.c_uint8)


class _ModuleDesc(ctypes.Structure):
    _fields_ = [("L", ctypes.c_uint32), ("K", ctypes.c_uint32), ("max_split", ctypes.c_uint32),
                ("w_max", ctypes.c_uint32), ("producer_mask", ctypes.c_uint32),
                ("chunk_layers", ctypes.c_void_p), ("f_ns", ctypes.c_void_p), ("b_ns", ctypes.c_void_p),
                ("act_kib", ctypes.c_void_p), ("p2p_ns", ctypes.c_void_p)]


class _ProblemDesc(ctypes.Structure):
    _fields_ = [("P", ctypes.c_uint32), ("n_modules", ctypes.c_uint32), ("m", ctypes.c_uint32),
                ("modules", ctypes.POINTER(_ModuleDesc)), ("inst_off", ctypes.c_void_p),
                ("inst_units", ctypes.c_void_p), ("budget_kib", ctypes.c_void_p)]


class _ModelInfo(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in ("P", "n_modules", "m", "n_max", "fbw", "record_stride",
                                                "group_lanes", "smem_per_block", "warps_per_block",
                                                "blocks_per_sm", "grid")] + [("makespan_bound", ctypes.c_uint64)]


class _CandBatch(ctypes.Structure):
    _fields_ = [("split", ctypes.c_void_p), ("n", ctypes.c_void_p), ("fwd_seq", ctypes.c_void_p),
                ("bwd_seq", ctypes.c_void_p), ("fb_bits", ctypes.c_void_p)]


class _SearchParams(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("rounds", ctypes.c_uint32), ("leaves", ctypes.c_uint32),
                ("rollouts", ctypes.c_uint32), ("threads", ctypes.c_int32), ("alpha", ctypes.c_double),
                ("beta", ctypes.c_double), ("memopt", ctypes.c_int32), ("policy", ctypes.c_int32),
                ("time_budget_ms", ctypes.c_double)]


class _SearchResult(ctypes.Structure):
    _fields_ = [("found", ctypes.c_int32), ("rounds_done", ctypes.c_uint32), ("makespan_ns", ctypes.c_uint64),
                ("score", ctypes.c_double), ("rollouts_scored", ctypes.c_uint64), ("tree_nodes", ctypes.c_uint64)]


class _Action(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in ("kind", "peer", "tag", "batch", "slot")]


ACTION_NAMES = ["fw_stage", "bw_stage", "isend", "irecv", "wait_isend", "wait_irecv"]


class _Winner(ctypes.Structure):
    _fields_ = [("found", ctypes.c_int32), ("rank", ctypes.c_int32), ("global_index", ctypes.c_uint64),
                ("makespan_ns", ctypes.c_uint64)]


@dataclass
class Winner:
    found: bool
    rank: int
    global_index: int
    makespan_ns: int


_lib = None


def lib():
    """Load libdip.so (built in-tree by paper_2504_14145_b200/build.py); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("DIP_LIB", LIB_PATH)     # an alternative in-tree build (kernel A/B runs)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run `python paper_2504_14145_b200/build.py` "
                           "(there is no CPU fallback for the scoring path)")
    L = ctypes.CDLL(path)
    st = ctypes.c_int
    vp = ctypes.c_void_p
    L.dip_load_cost_model.argtypes = [ctypes.POINTER(_ProblemDesc), ctypes.c_int, ctypes.POINTER(vp)]
    L.dip_model_free.argtypes = [vp]
    L.dip_model_get_info.argtypes = [vp, ctypes.POINTER(_ModelInfo)]
    L.dip_encode_candidates.argtypes = [vp, ctypes.POINTER(_CandBatch), ctypes.c_size_t, vp, ctypes.c_int]
    L.dip_workspace_create.argtypes = [vp, ctypes.c_size_t, ctypes.POINTER(vp)]
    L.dip_workspace_free.argtypes = [vp]
    L.dip_eval_schedules.argtypes = [vp, vp, vp, ctypes.c_size_t, vp, vp, vp]
    L.dip_interleave.argtypes = [vp, vp, vp, ctypes.c_size_t, vp, vp, vp, vp]
    L.dip_eval_orders.argtypes = [vp, vp, vp, vp, ctypes.c_size_t, vp, vp, vp, vp, vp, vp]
    L.dip_search.argtypes = [vp, vp, vp, ctypes.POINTER(_SearchParams), vp, vp, vp, ctypes.POINTER(_SearchResult), vp]
    L.dip_argmin.argtypes = [vp, vp, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, vp,
                             ctypes.POINTER(_Winner), vp]
    L.dip_encode_candidates_device.argtypes = [vp, ctypes.POINTER(_CandBatch), ctypes.c_size_t, vp, vp]
    L.dip_eval_host_view.argtypes = [vp, vp, ctypes.POINTER(_CandBatch), ctypes.c_size_t, vp, ctypes.c_uint64,
                                     ctypes.c_uint32, ctypes.c_uint32, vp, ctypes.POINTER(_Winner), vp]
    L.dip_eval_host.argtypes = [vp, vp, vp, ctypes.c_size_t, vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                vp, ctypes.POINTER(_Winner), vp]
    L.dip_pack_key.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                               ctypes.POINTER(ctypes.c_uint64)]
    L.dip_unpack_key.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(_Winner)]
    L.dip_timeline.argtypes = [vp, vp, vp, ctypes.c_size_t, vp, vp, vp, vp]
    L.dip_compile_plan.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp, ctypes.POINTER(ctypes.c_uint32)]
    L.dip_validate_plan.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.POINTER(ctypes.c_int32)]
    L.dip_set_strategies.argtypes = [vp, ctypes.c_uint32, vp, vp, vp, ctypes.c_uint32]
    L.dip_strategy_candidates.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, vp,
                                          ctypes.POINTER(ctypes.c_uint32)]
    L.dip_memopt.argtypes = [vp, vp, vp, vp, ctypes.c_size_t, vp, vp, vp, vp]
    L.dip_set_memopt_solver.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32]
    L.dip_memopt_stats.argtypes = [vp, vp, vp]
    L.dip_ubench_int.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(ctypes.c_double)]
    L.dip_comm_unique_id.argtypes = [vp]
    L.dip_comm_init.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    L.dip_comm_free.argtypes = [vp]
    for f in ("dip_load_cost_model", "dip_model_free", "dip_model_get_info", "dip_encode_candidates",
              "dip_workspace_create", "dip_workspace_free", "dip_eval_schedules", "dip_interleave", "dip_eval_orders",
              "dip_search",
              "dip_argmin",
              "dip_eval_host",
              "dip_comm_unique_id", "dip_comm_init", "dip_comm_free", "dip_pack_key", "dip_unpack_key",
              "dip_timeline", "dip_compile_plan", "dip_validate_plan",
              "dip_set_strategies", "dip_strategy_candidates", "dip_memopt", "dip_set_memopt_solver",
              "dip_memopt_stats", "dip_ubench_int", "dip_encode_candidates_device", "dip_eval_host_view"):
        getattr(L, f).restype = st
    L.dip_launch_count.restype = ctypes.c_uint64
    L.dip_launch_count.argtypes = []
    L.dip_status_str.restype = ctypes.c_char_p
    L.dip_status_str.argtypes = [st]
    L.dip_last_error.restype = ctypes.c_char_p
    L.dip_last_error.argtypes = []
    _lib = L
    return L


class DipError(RuntimeError):
    def __init__(self, code: int, where: str):
        L = lib()
        super().__init__(f"{where}: {L.dip_status_str(code).decode()} ({L.dip_last_error().decode()})")
        self.code = code


def _check(code: int, where: str):
    if code != DIP_OK:
        raise DipError(code, where)


def _ptr(a) -> int:
    if a is None:
        return 0
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _stream(stream) -> int:
    if stream is None:
        return 0
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def launch_count() -> int:
    return int(lib().dip_launch_count())


class Model:
    """dip_load_cost_model over a problem-like object (attributes P, m, modules[...] with
    L, K, max_split, w_max, producer_mask, f_ns, b_ns, act_kib, p2p_ns, chunk_layers;
    inst_off, inst_units, budget_kib)."""

    def __init__(self, pb, device: int = 0):
        L = lib()
        keep = []

        def arr(a, dt):
            x = np.ascontiguousarray(a, dt)
            keep.append(x)
            return x.ctypes.data

        mods = (_ModuleDesc * len(pb.modules))()
        for i, md in enumerate(pb.modules):
            mods[i] = _ModuleDesc(md.L, md.K, md.max_split, md.w_max, md.producer_mask,
                                  arr(md.chunk_layers, np.uint32) if md.chunk_layers is not None else None,
                                  arr(md.f_ns, np.uint32), arr(md.b_ns, np.uint32), arr(md.act_kib, np.uint32),
                                  arr(md.p2p_ns, np.uint32))
        units = np.ascontiguousarray(pb.inst_units, np.uint16)
        if units.size == 0:
            units = np.zeros(1, np.uint16)
        keep.append(units)
        d = _ProblemDesc(pb.P, len(pb.modules), pb.m, mods, arr(pb.inst_off, np.uint32), units.ctypes.data,
                         arr(pb.budget_kib, np.uint32))
        h = ctypes.c_void_p()
        _check(L.dip_load_cost_model(ctypes.byref(d), device, ctypes.byref(h)), "dip_load_cost_model")
        self.handle = h
        self.device = device
        inf = _ModelInfo()
        _check(L.dip_model_get_info(h, ctypes.byref(inf)), "dip_model_get_info")
        self.info = {k: getattr(inf, k) for k, _ in _ModelInfo._fields_}
        self.P = inf.P
        self.n_max = inf.n_max
        self.fbw = inf.fbw
        self.stride = inf.record_stride

    def refresh_info(self) -> dict:
        """re-read dip_model_get_info (dip_set_strategies may raise the makespan bound)"""
        inf = _ModelInfo()
        _check(lib().dip_model_get_info(self.handle, ctypes.byref(inf)), "dip_model_get_info")
        self.info = {k: getattr(inf, k) for k, _ in _ModelInfo._fields_}
        return self.info

    def encode(self, cands, out=None, threads: int = 0):
        """Pack host-view candidates (split, n, fwd, bwd, fb arrays) into records; returns `out`
        (a numpy uint8 array, or the given numpy array / pinned torch tensor)."""
        count = len(cands.n)
        if out is None:
            out = np.zeros(count * self.stride, np.uint8)
        arrs = [np.ascontiguousarray(getattr(cands, k)) for k in ("split", "n", "fwd", "bwd", "fb")]
        assert arrs[0].dtype == np.uint8 and arrs[1].dtype == np.uint32 and arrs[2].dtype == np.uint16
        assert arrs[4].dtype == np.uint32
        cb = _CandBatch(*[a.ctypes.data for a in arrs])
        _check(lib().dip_encode_candidates(self.handle, ctypes.byref(cb), count, _ptr(out), threads),
               "dip_encode_candidates")
        return out

    def set_strategies(self, menu, S: int = 10):
        """f3: per-layer strategy menu (f, b, act) arrays [n_strat, T] -> the GPU
        candidate table of every stage-pair type."""
        f, b, a = (np.ascontiguousarray(v, np.uint32) for v in menu)
        assert f.shape == b.shape == a.shape and f.ndim == 2
        _check(lib().dip_set_strategies(self.handle, f.shape[0], f.ctypes.data, b.ctypes.data, a.ctypes.data, S),
               "dip_set_strategies")
        self.S = S

    def strategy_candidates(self, module: int, layers: int, W: int):
        """the (F ns, B ns, mem KiB) candidates of one stage-pair type at width W"""
        out = np.zeros((16, 3), np.uint64)
        k = ctypes.c_uint32()
        _check(lib().dip_strategy_candidates(self.handle, module, layers, W, out.ctypes.data, ctypes.byref(k)),
               "dip_strategy_candidates")
        return [tuple(int(v) for v in out[x]) for x in range(k.value)]

    def close(self):
        if getattr(self, "handle", None):
            lib().dip_model_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Workspace:
    def __init__(self, model: Model, host_chunk: int = 0):
        h = ctypes.c_void_p()
        _check(lib().dip_workspace_create(model.handle, host_chunk, ctypes.byref(h)), "dip_workspace_create")
        self.handle = h
        self.model = model

    def close(self):
        if getattr(self, "handle", None):
            lib().dip_workspace_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Comm:
    """NCCL communicator owned by libdip (bootstrapped through torch.distributed)."""

    def __init__(self, uid: bytes, rank: int, world: int, device: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        _check(lib().dip_comm_init(buf, rank, world, device, ctypes.byref(h)), "dip_comm_init")
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().dip_comm_unique_id(buf), "dip_comm_unique_id")
        return bytes(buf)

    def close(self):
        if getattr(self, "handle", None):
            lib().dip_comm_free(self.handle)
            self.handle = None


def eval_schedules(model: Model, ws: Workspace, d_records, count: int, d_results, d_peaks=None, stream=None):
    """§8(a2)-(a6): score `count` device records (d_results: count x 24 B; d_peaks: [count, P] u32 or
    None) on `stream`, asynchronously; the fused argmin key is left in the workspace for argmin()."""
    _check(lib().dip_eval_schedules(model.handle, ws.handle, _ptr(d_records), count, _ptr(d_results),
                                    _ptr(d_peaks), _stream(stream)), "dip_eval_schedules")


def interleave(model: Model, ws: Workspace, d_records, count: int, d_results, d_peaks=None, d_orders=None,
               stream=None):
    """f1: DIP's dual-queue greedy on each record's split and priority orders; scores
    the built schedule (results as eval_schedules) and, with d_orders ([count][P][2 n_max] u16
    device), emits every rank's stage order (segment id | 0x8000 for backward, 0xFFFF padding)."""
    _check(lib().dip_interleave(model.handle, ws.handle, _ptr(d_records), count, _ptr(d_results),
                                _ptr(d_peaks), _ptr(d_orders), _stream(stream)), "dip_interleave")


def eval_orders(model: Model, ws: Workspace, d_records, d_orders, count: int, d_results, d_peaks=None, d_sel=None,
                d_start=None, d_end=None, stream=None):
    """Score schedules given as explicit per-rank orders (interleave's output format), optionally
    with an f3 selection (d_sel) and per-slot timelines (d_start / d_end [count][P][2 n_max] u64)."""
    _check(lib().dip_eval_orders(model.handle, ws.handle, _ptr(d_records), _ptr(d_orders), count, _ptr(d_sel),
                                 _ptr(d_results), _ptr(d_peaks), _ptr(d_start), _ptr(d_end), _stream(stream)),
           "dip_eval_orders")


def memopt(model: Model, ws: Workspace, d_records, count: int, d_sel, d_results, d_peaks=None, stream=None,
           d_orders=None):
    """f3: per-rank strategy selection (d_sel [count][P][2][n_max] u8 out) and the
    re-timed scores (results as eval_schedules); with d_orders the ranks' orders are those explicit
    per-rank orders (interleave's output) instead of the records' sequences + F/B bits."""
    _check(lib().dip_memopt(model.handle, ws.handle, _ptr(d_records), _ptr(d_orders), count, _ptr(d_sel),
                            _ptr(d_results), _ptr(d_peaks), _stream(stream)), "dip_memopt")


UBENCH_KINDS = ("IADD3", "VIMNMX", "ISETP+SEL", "SHFL+add", "IADD3+IADD3.X (u64 add)", "IMAD")


def ubench_int(device: int = 0) -> dict:
    """the integer-pipe microbenchmark: thread-level SASS instructions per second per kind"""
    out = {}
    for k, name in enumerate(UBENCH_KINDS):
        v, ms = ctypes.c_double(), ctypes.c_double()
        _check(lib().dip_ubench_int(k, device, ctypes.byref(v), ctypes.byref(ms)), "dip_ubench_int")
        out[name] = v.value
    return out


def set_memopt_solver(model: Model, gap_permille: int = 50, node_cap: int = 4096):
    """f3: the per-rank ILP's relative optimality gap (per mille) and B&B child budget."""
    _check(lib().dip_set_memopt_solver(model.handle, gap_permille, node_cap), "dip_set_memopt_solver")


def memopt_stats(ws: Workspace, stream=None) -> dict:
    """counters of the last memopt on ws: solved, certified (warm start within the gap at the root),
    searched (branch and bound), capped (node_cap reached), nodes (B&B children in total)"""
    out = np.zeros(5, np.uint64)
    _check(lib().dip_memopt_stats(ws.handle, out.ctypes.data, _stream(stream)), "dip_memopt_stats")
    return dict(zip(("solved", "certified", "searched", "capped", "nodes"), (int(v) for v in out)))


def search(model: Model, ws: Workspace, split, seed: int, rounds: int, leaves: int, rollouts: int,
           alpha: float = 1.0, beta: float = 0.5, threads: int = 0, stream=None, memopt: bool = False,
           policy: int = 0, time_budget_ms: float = 0.0) -> dict:
    """f2: MCTS over class orders for a fixed split with batched GPU rollouts (policy 1 /
    2: the random / depth-first exploration the paper compares against).
    Returns dict(found, makespan, score, trace, record (host bytes of the best rollout's split and
    priority orders), orders ([P, 2 n_max] its per-rank orders), ...)."""
    sp = np.ascontiguousarray(np.asarray(split, np.uint8).reshape(-1))
    prm = _SearchParams(seed & ((1 << 64) - 1), rounds, leaves, rollouts, threads, alpha, beta, 1 if memopt else 0,
                        policy, time_budget_ms)
    out = _SearchResult()
    rec = np.zeros(model.stride, np.uint8)
    ords = np.zeros((model.P, 2 * model.n_max), np.uint16)
    trace = np.zeros(rounds, np.float64)
    _check(lib().dip_search(model.handle, ws.handle, sp.ctypes.data, ctypes.byref(prm), rec.ctypes.data,
                            ords.ctypes.data, trace.ctypes.data, ctypes.byref(out), _stream(stream)), "dip_search")
    return dict(found=bool(out.found), makespan=out.makespan_ns, score=out.score, trace=trace, record=rec,
                orders=ords, rounds_done=out.rounds_done, scored=out.rollouts_scored, tree_nodes=out.tree_nodes)


def timeline(model: Model, ws: Workspace, d_records, count: int, d_results, d_start, d_end, stream=None):
    """eval_schedules + per-slot start / end times ([count][P][2*n_max] u64 device buffers)."""
    _check(lib().dip_timeline(model.handle, ws.handle, _ptr(d_records), count, _ptr(d_results), _ptr(d_start),
                              _ptr(d_end), _stream(stream)), "dip_timeline")


def compile_plan(model: Model, record, start, end, orders=None):
    """f4: per-rank action lists of one schedule. record: host uint8[stride];
    start / end: host uint64 [P, 2*n_max]; orders: None (the record's sequences + bits) or host
    [P, 2*n_max] u16 per-rank orders (interleave's output). Returns (actions, rank_off, n_messages)."""
    rec = np.ascontiguousarray(record, np.uint8)
    od = None if orders is None else np.ascontiguousarray(orders, np.uint16)
    st = np.ascontiguousarray(start, np.uint64)
    en = np.ascontiguousarray(end, np.uint64)
    off = np.zeros(model.P + 1, np.uint32)
    nmsg = ctypes.c_uint32()
    cap = 1 << 16
    while True:
        acts = np.zeros((cap, 5), np.uint32)
        code = lib().dip_compile_plan(model.handle, rec.ctypes.data, None if od is None else od.ctypes.data,
                                      st.ctypes.data, en.ctypes.data, acts.ctypes.data, cap, off.ctypes.data,
                                      ctypes.byref(nmsg))
        if code == 4 and off[-1] > cap:   # DIP_ERANGE: grow
            cap = int(off[-1])
            continue
        _check(code, "dip_compile_plan")
        return acts[: off[-1]], off, nmsg.value


def validate_plan(model: Model, record, acts, off, orders=None):
    """Discrete-event execution of a plan -> (ok, stage start times [P, 2*n_max])."""
    rec = np.ascontiguousarray(record, np.uint8)
    od = None if orders is None else np.ascontiguousarray(orders, np.uint16)
    a = np.ascontiguousarray(acts, np.uint32)
    o = np.ascontiguousarray(off, np.uint32)
    st = np.zeros((model.P, 2 * model.n_max), np.uint64)
    ok = ctypes.c_int32()
    _check(lib().dip_validate_plan(model.handle, rec.ctypes.data, None if od is None else od.ctypes.data,
                                   a.ctypes.data, o.ctypes.data, st.ctypes.data, ctypes.byref(ok)),
           "dip_validate_plan")
    return bool(ok.value), st


def argmin(model: Model, ws: Workspace, count: int, shard_stride: Optional[int] = None, rank: int = 0,
           world: int = 1, comm: Optional[Comm] = None, stream=None) -> Winner:
    """§8(a7): the winner of the last scoring call -- lowest (makespan, global index) among status-OK
    candidates, across ranks through one NCCL allreduce when `comm` is given. Synchronous."""
    w = _Winner()
    _check(lib().dip_argmin(model.handle, ws.handle, count, shard_stride if shard_stride is not None else count,
                            rank, world, comm.handle if comm else None, ctypes.byref(w), _stream(stream)),
           "dip_argmin")
    return Winner(bool(w.found), w.rank, w.global_index, w.makespan_ns)


def eval_host(model: Model, ws: Workspace, h_records, count: int, h_results=None, shard_stride: Optional[int] = None,
              rank: int = 0, world: int = 1, comm: Optional[Comm] = None, stream=None) -> Winner:
    """End to end from host records (pinned for overlap): chunked H2D overlapped with scoring on two
    streams, then argmin(). h_results (host, count x 24 B) may be None. Synchronous."""
    w = _Winner()
    _check(lib().dip_eval_host(model.handle, ws.handle, _ptr(h_records), count, _ptr(h_results),
                               shard_stride if shard_stride is not None else count, rank, world,
                               comm.handle if comm else None, ctypes.byref(w), _stream(stream)), "dip_eval_host")
    return Winner(bool(w.found), w.rank, w.global_index, w.makespan_ns)


def _batch(arrs):
    """the five host-view arrays (numpy arrays or tensors: split u8, n u32, fwd u16, bwd u16, fb u32)"""
    return _CandBatch(*[_ptr(a) for a in arrs])


def encode_device(model: Model, d_view, count: int, d_out, stream=None):
    """§8(b) device mode: pack candidates whose host-view arrays (split, n, fwd, bwd, fb) are already
    on the device (tensors) into device records d_out."""
    cb = _batch(d_view)
    _check(lib().dip_encode_candidates_device(model.handle, ctypes.byref(cb), count, _ptr(d_out), _stream(stream)),
           "dip_encode_candidates_device")


def eval_host_view(model: Model, ws: Workspace, h_view, count: int, h_results=None, shard_stride: Optional[int] = None,
                   rank: int = 0, world: int = 1, comm: Optional[Comm] = None, stream=None) -> Winner:
    """End to end from the candidates' host view (pinned split, n, fwd, bwd, fb arrays / tensors):
    chunked H2D -> device encode -> scoring -> results D2H (h_results may be None) -> argmin."""
    cb = _batch(h_view)
    w = _Winner()
    _check(lib().dip_eval_host_view(model.handle, ws.handle, ctypes.byref(cb), count, _ptr(h_results),
                                    shard_stride if shard_stride is not None else count, rank, world,
                                    comm.handle if comm else None, ctypes.byref(w), _stream(stream)),
           "dip_eval_host_view")
    return Winner(bool(w.found), w.rank, w.global_index, w.makespan_ns)


def pack_key(makespan_ns: int, rank: int, local: int, shard_stride: int, world: int) -> int:
    """Cross-rank argmin key (host side of dip_argmin's packed allreduce)."""
    k = ctypes.c_uint64()
    _check(lib().dip_pack_key(makespan_ns, rank, local, shard_stride, world, ctypes.byref(k)), "dip_pack_key")
    return k.value


def unpack_key(key: int, shard_stride: int, world: int) -> Winner:
    """Inverse of pack_key (UINT64_MAX -> not found)."""
    w = _Winner()
    _check(lib().dip_unpack_key(key, shard_stride, world, ctypes.byref(w)), "dip_unpack_key")
    return Winner(bool(w.found), w.rank, w.global_index, w.makespan_ns)


def results_view(host_bytes) -> np.ndarray:
    """View a host copy of dip_result[count] (uint8 bytes) as a structured numpy array."""
    a = np.asarray(host_bytes)
    return a.view(RESULT_DTYPE)
