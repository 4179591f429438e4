"""The oracle against the worked examples printed in PAPER.md and SPEC.md, kept as cited text
fixtures under tests/golden/ (each file names its source lines)."""
import os
from fractions import Fraction

import numpy as np
import yaml

import oracle
from gen import Module, Problem
from tests import helpers as H

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GB = 1 << 20


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return yaml.safe_load(f)


def test_every_fixture_cites_its_source():
    for fn in os.listdir(GOLD):
        d = load(fn)
        assert d.get("source"), fn


def test_chunking_and_split():
    g = load("spec_chunking_and_split.yaml")
    for c in g["chunking"]:
        assert oracle.chunk_layers(c["L"], c["P"], c["K"]) == c["layers"]
    for c in g["split"]:
        assert oracle.split_sizes(c["N"], c["M"]) == c["sizes"]


def test_1f1b_bubble():
    g = load("spec_1f1b_bubble.yaml")
    pb = H.uniform_problem(g["P"], g["m"], 1, 2)
    cs = H.candidates_from_orders(pb, [[1] * g["m"]], [H.one_f_one_b(g["P"], g["m"])])
    r = oracle.evaluate(pb, cs)
    assert r.bubble[0] == float(Fraction(g["bubble_num"], g["bubble_den"]))
    assert round(r.bubble[0] * 100, 2) == g["bubble_pct_printed"]


def test_s2_2_stage_imbalance():
    g = load("paper_s2_2_stage_imbalance.yaml")
    # the min-max partition of SURVEY App. A.3 (6 x 10 ViT | 4 ViT + 4 LM | 3 x 6 LM | 6 x 7 LM),
    # in units of 0.25 ms of forward (F:B = 1:2): ViT layer 9 units, LM layer 14 units
    vit_u, lm_u = round(g["vit_layer_fb_ms"] / 0.75), round(g["lm_layer_fb_ms"] / 0.75)
    chunks = [10 * vit_u] * 6 + [4 * vit_u + 4 * lm_u] + [6 * lm_u] * 3 + [7 * lm_u] * 6
    assert len(chunks) == g["stages"]
    fb_ms = [c * 0.75 for c in chunks]
    assert min(fb_ms) == g["stage_min_ms"] and max(fb_ms) == g["stage_max_ms"]
    assert round((max(fb_ms) - min(fb_ms)) / min(fb_ms) * 100, 1) == g["variation_pct"]
    m = g["microbatches"]
    md = Module("mixed", sum(chunks), 1, 1, 1, 0, *H.table(1, {1: (250_000, 500_000, 1, 0)}),
                chunk_layers=np.array(chunks, np.uint32))
    pb = Problem("s22", g["stages"], m, [md], np.arange(m + 1, dtype=np.uint32), np.ones(m, np.uint16),
                 np.full(g["stages"], 1 << 31, np.uint32))
    cs = H.candidates_from_orders(pb, [[1] * m], [H.one_f_one_b(g["stages"], m)])
    r = oracle.evaluate(pb, cs)
    assert abs(r.bubble[0] * 100 - g["bubble_pct"]) <= g["bubble_tolerance_pct"]


def test_memory_optimisation_examples():
    g = load("spec_memory_optimisation.yaml")
    for c in g["candidates"]:
        st = c["strategies"]
        got = oracle.mem_candidates([s["f"] for s in st], [s["b"] for s in st], [s["mem_gb"] * GB for s in st],
                                    layers=c["layers"], S=c["S"])
        assert [[f + b, m // GB] for f, b, m in got] == c["expected"]
    sel = g["selection"]
    pair = sel["pair"]
    for case in sel["cases"]:
        md = Module("m", 1, 1, 1, 1, 0, *H.table(1, {1: (pair[0]["f"], pair[0]["b"], pair[0]["mem_gb"] * GB, 0)}))
        pb = Problem("pair", 1, 1, [md], np.array([0, 1], np.uint32), np.ones(1, np.uint16),
                     np.array([case["budget_gb"] * GB], np.uint32))
        menu = (np.array([[0, s["f"]] for s in pair], np.uint32), np.array([[0, s["b"]] for s in pair], np.uint32),
                np.array([[0, s["mem_gb"] * GB] for s in pair], np.uint32))
        cs = H.candidates_from_orders(pb, [[1]], [[[("F", 0), ("B", 0)]]])
        sel_out, r = oracle.memopt(pb, cs, menu, S=10)
        assert int(r.makespan[0]) == case["latency_ms"] and int(r.peaks[0, 0]) == case["mem_gb"] * GB
