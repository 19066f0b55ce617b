"""The byte counter behind every GB/s figure bench.py reports (CPU only).

bench.step_bytes is pinned to SURVEY.md 8(d) d5's table (computed there from the
BASELINE.json configs, not by this code) and bench.kv_cache_bytes to SPEC.md:331's
worked example (P12: 10 entries, 1 layer, 1 KV head, d 4, 8-byte elements -> 640 B)."""
import json
import os

import pytest

import bench
from paper_2510_17777_b200 import inputs as gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _qoi(wl):  # q in, out, idx: on top of d5's K/V bytes in bench's totals
    return wl.B * wl.H * wl.d * 2 + wl.B * wl.H * wl.d * 4 + wl.B * wl.Hkv * wl.k * 4


@pytest.mark.parametrize("case", GOLD["d5_step_bytes"]["cases"], ids=lambda c: c["config"])
def test_step_bytes_match_survey_d5(case):
    wl = gen.CONFIGS[case["config"]]
    b = bench.step_bytes(wl)
    assert abs((b["total"] - _qoi(wl)) / 1e6 - case["step_MB"]) <= case["tol_MB"]
    assert abs((b["decode"] - _qoi(wl)) / 1e6 - case["steady_MB"]) <= case["tol_MB"]


def test_step_bytes_components():
    wl = gen.CONFIGS["long-video"]
    b = bench.step_bytes(wl)
    row = wl.d * 2
    T = wl.vb + wl.t_after
    # scored visual K = 32 MiB exactly (d5), selected K+V of k rows, text K+V of T rows
    assert wl.B * wl.Hkv * wl.nv * row == 32 * 2 ** 20
    assert b["total"] - b["decode"] == wl.B * wl.Hkv * wl.nv * row
    # the fused kernel does not re-read the kept K rows (their logits stay on chip)
    assert b["total"] - b["fused"] == wl.B * wl.Hkv * wl.k * row
    assert b["score"] == wl.B * wl.Hkv * (wl.nv + T) * row + wl.B * wl.H * row


def test_kv_cache_bytes_spec_example():
    p = GOLD["P12_bytes"]
    assert bench.kv_cache_bytes(p["entries"], p["layers"], p["kv_heads"], p["d"], p["elem_bytes"]) == p["bytes"]
