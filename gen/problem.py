"""Seeded synthetic problems (configs, per-layer cost tables, batch workloads).

INPUT GENERATION ONLY. This module is shared by the oracle tests and the CUDA
path, so it holds none of the hot path's arithmetic: no sub-microbatch split,
no cost lookup, no timing, no memory scan.
It builds the *inputs* of `dip_load_cost_model` (§3.2 step 1,
"metadata ... token counts, number of images"):

* the model structure: P ranks, modules with L_i layers, K_i segments
  (P:450-459), M_max,i (the sub-microbatch menu, reading R-2);
* per-layer integer tables T_i[W] = {F ns, B ns, act KiB, p2p ns} from the
  simulator's operator latency model max{a_fop N_fop/F, ...},
  reduced to the FLOP term (reading R-8/R-20);
* the batch: per (microbatch b, module i) instance work units, packed greedily
  into 8192-token microbatches with 169 tokens per image;
* per-rank activation budgets (capacity M minus static memory).

Seeds: seed = 250414145 + config_index; sub-streams splitmix64(seed, tag).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

SEED_BASE = 250414145
CONFIG_NAMES = ["toy", "12B", "37B", "T2V", "94B"]

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """splitmix64 finaliser (same constants as gen/dip_gen.c)."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def substream(seed: int, tag: str) -> int:
    h = seed
    for ch in tag.encode():
        h = splitmix64(h ^ ch)
    return h


@dataclasses.dataclass
class Module:
    name: str
    L: int                 # layers
    K: int                 # pipeline segments
    max_split: int         # M_max: candidate chooses M in [1, min(N, M_max)] (R-2)
    w_max: int             # table covers W in [0, w_max]
    producer_mask: int     # modules whose outputs feed this one (R-5)
    f_ns: np.ndarray       # uint32 [w_max+1] per-layer forward latency
    b_ns: np.ndarray       # uint32 [w_max+1] per-layer backward latency
    act_kib: np.ndarray    # uint32 [w_max+1] per-layer activation KiB
    p2p_ns: np.ndarray     # uint32 [w_max+1] boundary transfer latency
    chunk_layers: Optional[np.ndarray] = None   # optional uint32 [P*K] override


@dataclasses.dataclass
class Problem:
    name: str
    P: int
    m: int
    modules: List[Module]
    inst_off: np.ndarray     # uint32 [m*nmod+1], b-major
    inst_units: np.ndarray   # uint16 per-instance work units (R-21)
    budget_kib: np.ndarray   # uint32 [P]
    seed: int = 0

    @property
    def nmod(self) -> int:
        return len(self.modules)

    @property
    def n_max(self) -> int:
        return self.m * sum(md.max_split * md.K for md in self.modules)

    @property
    def fbw(self) -> int:
        return max(1, (2 * self.n_max + 31) // 32)

    def n_inst(self) -> np.ndarray:
        """N_{b,i} = instance count per (microbatch, module), shape [m, nmod]."""
        return np.diff(self.inst_off.astype(np.int64)).reshape(self.m, self.nmod)

    def seg_base(self) -> np.ndarray:
        """Segment-id base per (b, i): id(b,i,j,k) = base + j*K_i + k."""
        per = [md.max_split * md.K for md in self.modules]
        base = np.zeros((self.m, self.nmod), dtype=np.int64)
        acc = 0
        for b in range(self.m):
            for i in range(self.nmod):
                base[b, i] = acc
                acc += per[i]
        return base

    def seg_decode(self) -> np.ndarray:
        """[n_max, 4] rows (b, i, j, k) for every segment id."""
        out = np.zeros((self.n_max, 4), dtype=np.int64)
        base = self.seg_base()
        for b in range(self.m):
            for i, md in enumerate(self.modules):
                for j in range(md.max_split):
                    for k in range(md.K):
                        out[base[b, i] + j * md.K + k] = (b, i, j, k)
        return out

    def consumer_mask(self, i: int) -> int:
        return sum(1 << c for c, md in enumerate(self.modules) if (md.producer_mask >> i) & 1)


# ---------------------------------------------------------------------------
# Per-layer tables from the operator latency model
# ---------------------------------------------------------------------------
F_DEV = 989e12        # H800-class dense BF16 FLOP/s (the paper's testbed)
ALPHA = 0.5           # alpha_fop efficiency factor
OVERHEAD_NS = 20_000  # per-layer fixed cost (small-batch under-utilisation)
NET_BPS = 200e9       # NVLink 200 GB/s


@dataclasses.dataclass
class Arch:
    """Transformer dimensions (Table)."""
    layers: int
    h: int
    ffn: int
    heads: int
    groups: int
    gated: bool    # SwiGLU (3 matrices) vs GELU MLP (2)


ARCH = {
    "vit5b": Arch(63, 1792, 15360, 16, 16, False),
    "vit22b": Arch(48, 6144, 24576, 48, 48, False),
    "llama3_8b": Arch(32, 4096, 14336, 32, 8, True),
    "qwen2_32b": Arch(64, 5120, 27648, 40, 8, True),
    "qwen2_72b": Arch(80, 8192, 29568, 64, 8, True),
    "dit30b": Arch(48, 6144, 24576, 48, 48, False),
}


def layer_params(a: Arch) -> float:
    kv = a.h * a.groups // a.heads
    attn = a.h * (a.h + 2 * kv) + a.h * a.h
    mlp = (3 if a.gated else 2) * a.h * a.ffn
    return float(attn + mlp)


def make_tables(a: Arch, w_max: int, tokens_per_unit: float, attn_span, tp: int,
                conv_flops_per_unit: float = 0.0):
    """Integer per-layer tables for W = 0..w_max (W = 0 -> all zeros).

    tokens s = tokens_per_unit * W; FLOPs_fwd = 2*params*s + 4*s*ctx*h where ctx
    is the attention span (per image for ViT, the whole sequence otherwise);
    B = 2*F in FLOPs; act = 34*s*h bytes / TP rounded up to KiB
    (R-9); p2p = 2*s*h bytes / TP over 200 GB/s (R-7). All rounded up once (R-8).
    """
    n = w_max + 1
    f = np.zeros(n, np.uint32)
    b = np.zeros(n, np.uint32)
    act = np.zeros(n, np.uint32)
    p2p = np.zeros(n, np.uint32)
    prm = layer_params(a)
    for w in range(1, n):
        s = tokens_per_unit * w
        ctx = attn_span(w, s)
        flops = 2.0 * prm * s + 4.0 * s * ctx * a.h + conv_flops_per_unit * w
        fns = math.ceil(flops / tp / (ALPHA * F_DEV) * 1e9) + OVERHEAD_NS
        bns = math.ceil(2.0 * flops / tp / (ALPHA * F_DEV) * 1e9) + OVERHEAD_NS
        f[w] = fns
        b[w] = bns
        act[w] = math.ceil(34.0 * s * a.h / tp / 1024.0)
        p2p[w] = math.ceil(2.0 * s * a.h / tp / NET_BPS * 1e9)
    return f, b, act, p2p


# ---------------------------------------------------------------------------
# Workload samplers
# ---------------------------------------------------------------------------
IMG_TOKENS = 169       # P:769 "one image into 169 patch tokens"
SEQ_TOKENS = 8192      # P:770 context length
MAX_IMAGES = SEQ_TOKENS // IMG_TOKENS   # 48


def _sample_vlm_item(rng: np.random.Generator, video: bool):
    """One sample -> (list of vision instance units, text tokens)."""
    u = rng.random()
    if video and u < 0.25:
        dur = math.exp(rng.uniform(math.log(1.0), math.log(16.0)))
        frames = max(2, min(32, int(round(2 * dur))))      # 2 frames/s, 1 unit = 1 frame
        return [frames], int(rng.integers(16, 129))
    u = rng.random()
    if u < 0.45:     # caption pair (LAION-like, ~16.4 tokens/image)
        return [1], int(rng.integers(8, 26))
    if u < 0.80:     # interleaved document (OBELICS-like, 0.4..3115 tokens/image)
        k = int(rng.integers(1, 11))
        per = math.exp(rng.uniform(math.log(0.4), math.log(3115.0)))
        return [1] * k, max(1, int(per * k))
    if u < 0.90:     # QA
        return [1], int(rng.integers(64, 513))
    return [], int(rng.integers(512, 4097))   # text only


def _pack_vlm(rng, m: int, video: bool, llm_unit_tokens: int = 64):
    """First-fit packing to 8192 tokens; returns per-mb (vision units, llm units)."""
    mbs = []
    while len(mbs) < m:
        vis, toks = [], 0
        tries = 0
        while tries < 64:
            units, text = _sample_vlm_item(rng, video)
            need = sum(units) * IMG_TOKENS + text
            if need > SEQ_TOKENS:
                tries += 1
                continue
            if toks + need > SEQ_TOKENS or sum(vis) + sum(units) > MAX_IMAGES:
                tries += 1
                if toks > SEQ_TOKENS // 2:
                    break
                continue
            vis.extend(units)
            toks += need
        llm_units = max(1, -(-toks // llm_unit_tokens))
        mbs.append((vis, [llm_units]))
    return mbs


def _pack_t2v(rng, m: int):
    """Clips of log-uniform [1, 16] s; first-fit <= 8 clips and <= 16 s per mb."""
    mbs = []
    while len(mbs) < m:
        clips = []   # (seconds_units, caption_units)
        secs = 0
        tries = 0
        while tries < 64 and len(clips) < 8:
            d = math.exp(rng.uniform(0.0, math.log(16.0)))
            su = max(1, math.ceil(d))
            cap = int(rng.integers(16, 257))
            if secs + su > 16:
                tries += 1
                if secs >= 12:
                    break
                continue
            clips.append((su, -(-cap // 16)))
            secs += su
        if clips:
            mbs.append(clips)
    return mbs


def _budgets(P: int, capacity_gb: float, static_bytes_per_rank: np.ndarray) -> np.ndarray:
    cap = capacity_gb * (1 << 30)
    return np.maximum(0, (cap - static_bytes_per_rank) // 1024).astype(np.uint32)


def _chunk_params(md_layers_per_chunk: List[np.ndarray], params: List[float], tp: int, P: int):
    """Static bytes per rank: 16 B/param (weights+grads+Adam, P:802 context) / TP."""
    out = np.zeros(P)
    for lay, prm in zip(md_layers_per_chunk, params):
        Kp = len(lay) // P
        for k in range(Kp):
            for r in range(P):
                out[r] += 16.0 * lay[k * P + r] * prm / tp
    return out


def _default_chunks(L: int, P: int, K: int) -> np.ndarray:
    C = P * K
    q, rem = divmod(L, C)
    return np.array([q + (1 if c < rem else 0) for c in range(C)], dtype=np.int64)


def make_problem(name: str) -> Problem:
    """Build the seeded synthetic problem of one of the five BASELINE.json configs."""
    idx = CONFIG_NAMES.index(name)
    seed = SEED_BASE + idx
    rng = np.random.default_rng(substream(seed, "workload") & 0xFFFFFFFFFFFF)

    if name == "toy":
        P, m = 4, 4
        wv, wl = 16, 128
        w = np.arange(wv + 1, dtype=np.uint64)
        vf = np.where(w > 0, 100 * w + 50, 0).astype(np.uint32)
        wl_ = np.arange(wl + 1, dtype=np.uint64)
        lf = np.where(wl_ > 0, 10 * wl_ + 100, 0).astype(np.uint32)
        vit = Module("vit", 8, 1, 2, wv, 0, vf, 2 * vf, (10 * w).astype(np.uint32),
                     np.zeros(wv + 1, np.uint32))
        llm = Module("llm", 8, 1, 1, wl, 1, lf, 2 * lf, (10 * wl_).astype(np.uint32),
                     np.zeros(wl + 1, np.uint32))
        units, off = [], [0]
        for b in range(m):
            while True:
                imgs, toks = 0, 0
                for _ in range(8):
                    kind = int(rng.integers(0, 3))
                    if kind == 0:
                        toks += int(rng.integers(64, 257))
                    else:
                        imgs += kind
                        toks += kind * IMG_TOKENS + int(rng.integers(8, 33))
                if 2 <= imgs <= 16:
                    break
            units += [1] * imgs
            off.append(len(units))
            units.append(-(-toks // 64))
            off.append(len(units))
        return Problem(name, P, m, [vit, llm], np.array(off, np.uint32),
                       np.array(units, np.uint16), np.full(P, 1 << 30, np.uint32), seed)

    if name in ("12B", "37B", "94B"):
        if name == "12B":
            P, m, tp = 8, 16, 4
            va, la, K_llm, cap_gb = ARCH["vit5b"], ARCH["llama3_8b"], 4, 80.0
        elif name == "37B":
            P, m, tp = 8, 32, 8
            va, la, K_llm, cap_gb = ARCH["vit5b"], ARCH["qwen2_32b"], 2, 80.0
        else:
            P, m, tp = 32, 64, 8
            va, la, K_llm, cap_gb = ARCH["vit22b"], ARCH["qwen2_72b"], 2, 80.0
        video = name != "12B"
        mbs = _pack_vlm(rng, m, video)
        wv = MAX_IMAGES
        wl = SEQ_TOKENS // 64 + 1
        vt = make_tables(va, wv, IMG_TOKENS, lambda w, s: IMG_TOKENS, tp)
        lt = make_tables(la, wl, 64, lambda w, s: s, tp)
        vit = Module("vit", va.layers, 1, 4, wv, 0, *vt)
        llm = Module("llm", la.layers, K_llm, 1, wl, 1, *lt)
        units, off = [], [0]
        for vis, lu in mbs:
            units += vis
            off.append(len(units))
            units += lu
            off.append(len(units))
        mods = [vit, llm]
        stat = _chunk_params([_default_chunks(md.L, P, md.K) for md in mods],
                             [layer_params(va), layer_params(la)], tp, P)
        return Problem(name, P, m, mods, np.array(off, np.uint32), np.array(units, np.uint16),
                       _budgets(P, CAPACITY_GB[name], stat), seed)

    if name == "T2V":
        P, m, tp = 16, 32, 8
        ta, da = ARCH["qwen2_32b"], ARCH["dit30b"]
        mbs = _pack_t2v(rng, m)
        wt, wv, wd = 128, 16, 16
        tt = make_tables(ta, wt, 16, lambda w, s: s, tp)
        # VAE: 16 conv blocks; cost per second of video (assumed, R-22)
        vae_arch = Arch(16, 512, 2048, 8, 8, False)
        vt = make_tables(vae_arch, wv, 4096, lambda w, s: 64, tp, conv_flops_per_unit=4.0e12)
        dt = make_tables(da, wd, 1024, lambda w, s: s, tp)
        text = Module("text_enc", ta.layers, 1, 1, wt, 0, *tt)
        vae = Module("vae", 16, 1, 4, wv, 0, *vt)
        dit = Module("dit", da.layers, 2, 2, wd, 0b011, *dt)
        units, off = [], [0]
        for clips in mbs:
            units += [c for _, c in clips]
            off.append(len(units))
            units += [s for s, _ in clips]
            off.append(len(units))
            units += [s for s, _ in clips]
            off.append(len(units))
        mods = [text, vae, dit]
        stat = _chunk_params([_default_chunks(md.L, P, md.K) for md in mods],
                             [layer_params(ta), layer_params(vae_arch), layer_params(da)], tp, P)
        return Problem(name, P, m, mods, np.array(off, np.uint32), np.array(units, np.uint16),
                       _budgets(P, CAPACITY_GB[name], stat), seed)
    raise KeyError(name)


# Memory capacity M per rank in GB available to weights+activations: the 80 GB of
# an H800 minus unmodelled runtime buffers, set so that a minority of the generated
# candidates exceed it (5-25% OOM); bench.py reports the exact status histogram.
CAPACITY_GB = {"12B": 24.0, "37B": 34.0, "T2V": 44.0, "94B": 65.0}


def problem_arrays(pb: Problem):
    """Flatten a Problem into the plain arrays the C entry points take."""
    nm = pb.nmod
    mods = pb.modules
    L = np.array([md.L for md in mods], np.uint32)
    K = np.array([md.K for md in mods], np.uint32)
    ms = np.array([md.max_split for md in mods], np.uint32)
    wm = np.array([md.w_max for md in mods], np.uint32)
    pm = np.array([md.producer_mask for md in mods], np.uint32)
    toff = np.zeros(nm + 1, np.uint32)
    for i, md in enumerate(mods):
        toff[i + 1] = toff[i] + md.w_max + 1
    tf = np.concatenate([md.f_ns for md in mods]).astype(np.uint32)
    tb = np.concatenate([md.b_ns for md in mods]).astype(np.uint32)
    ta = np.concatenate([md.act_kib for md in mods]).astype(np.uint32)
    tp = np.concatenate([md.p2p_ns for md in mods]).astype(np.uint32)
    coff = np.zeros(nm + 1, np.uint32)
    cl = []
    for i, md in enumerate(mods):
        if md.chunk_layers is not None:
            arr = np.asarray(md.chunk_layers, np.uint32)
        else:
            arr = np.zeros(0, np.uint32)
        cl.append(arr)
        coff[i + 1] = coff[i] + len(arr)
    chunk = np.concatenate(cl).astype(np.uint32) if cl else np.zeros(0, np.uint32)
    return dict(L=L, K=K, max_split=ms, w_max=wm, producer_mask=pm, tab_off=toff,
                tab_f=tf, tab_b=tb, tab_act=ta, tab_p2p=tp, chunk_off=coff, chunk_layers=chunk)


# ---------------------------------------------------------------------------
# Per-layer memory-strategy menu (f3, §5.3; R-37)
# ---------------------------------------------------------------------------
N_STRAT = 3
# strategy c: backward latency saved (in units of the layer's forward latency) and activation
# growth factor, relative to the base tables (strategy 0 = the most memory-efficient scheme,
# the one every other row uses): 0 keeps the base recomputation, 1 keeps the MLP
# activations (no MLP recompute), 2 keeps everything (no recompute at all).
STRAT_SAVE = ((0, 1), (1, 4), (2, 5))        # fraction num/den of F saved in B
STRAT_GROW = ((1, 1), (3, 2), (9, 4))        # activation x num/den


def strategy_menu(pb: Problem):
    """(f, b, act) uint32 arrays [N_STRAT, T] aligned with problem_arrays' tables (T = sum of
    w_max_i + 1): per-layer F ns, B ns and activation KiB of each strategy. Input data only."""
    a = problem_arrays(pb)
    T = len(a["tab_f"])
    f = np.zeros((N_STRAT, T), np.uint32)
    b = np.zeros((N_STRAT, T), np.uint32)
    act = np.zeros((N_STRAT, T), np.uint32)
    tf = a["tab_f"].astype(np.uint64)
    tb = a["tab_b"].astype(np.uint64)
    ta = a["tab_act"].astype(np.uint64)
    for c in range(N_STRAT):
        (sn, sd), (gn, gd) = STRAT_SAVE[c], STRAT_GROW[c]
        f[c] = tf
        b[c] = tb - (tf * sn) // sd
        act[c] = (ta * gn + gd - 1) // gd
    return f, b, act
