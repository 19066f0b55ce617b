"""Pins of oracle.question_attention (the question chunk's
attention output) against things other than itself (-m "not gpu"):

  P16a  the last question row sees the whole sequence: equals the C decode oracle
        dense_attn (o_dense_attn, independent code) for q = q[:, n_q-1];
  P16b  VISUAL_ONLY equals dense_attn on a cache cut down to the visual rows;
  P16c  brute force on a tiny case with math.exp loops (causal limit per row);
  P16d  causality: rows past L - n_q + r do not change row r, rows inside do;
  P16e  a constant V gives that constant (the weights sum to one), and lse_in
        shifted by c scales the output by exp(-c).
A wrong causal limit, a dropped GQA mapping (h -> h // g), K/V transposed or the
LSE taken over the wrong range fails at least one of them.
"""
import math

import numpy as np
import pytest
import torch

from paper_2510_17777_b200 import inputs as gen


def _case(B=2, n_q=5, H=6, Hkv=2, d=16, vb=4, nv=40, ta=9, seed=1):
    wl = gen.DecodeWorkload("qa", B, H, Hkv, d, vb, nv, ta, 8, n_q, 16,
                            seq_lens=[vb + nv + ta - b for b in range(B)])
    return wl, gen.make_decode_inputs(wl, seed=seed)


def test_P16a_last_row_equals_dense_decode(orc):
    wl, x = _case()
    out, lse, _ = orc.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv)
    o2, l2 = orc.dense_attn(x["q"][:, -1].contiguous(), x["K"], x["V"], x["seq_len"])
    assert np.allclose(out[:, -1], o2, atol=1e-12, rtol=0)
    assert np.allclose(lse[:, -1], l2, atol=1e-12, rtol=0)


def test_P16b_visual_only_equals_dense_on_visual_rows(orc):
    wl, x = _case(seed=2)
    out, lse, _ = orc.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv,
                                         flags=orc.VISUAL_ONLY)
    Kv = x["K"][:, :, wl.vb:wl.vb + wl.nv].contiguous()
    Vv = x["V"][:, :, wl.vb:wl.vb + wl.nv].contiguous()
    nvs = torch.full((wl.B,), wl.nv, dtype=torch.int32)
    for r in range(wl.n_q):
        o2, l2 = orc.dense_attn(x["q"][:, r].contiguous(), Kv, Vv, nvs)
        assert np.allclose(out[:, r], o2, atol=1e-12, rtol=0)
        assert np.allclose(lse[:, r], l2, atol=1e-12, rtol=0)


def test_P16c_bruteforce_tiny(orc):
    wl, x = _case(B=1, n_q=3, H=4, Hkv=2, d=4, vb=2, nv=5, ta=4, seed=3)
    out, lse, absm = orc.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv)
    q, K, V = x["q"].double(), x["K"].double(), x["V"].double()
    L = int(x["seq_len"][0])
    g = wl.H // wl.Hkv
    for r in range(wl.n_q):
        for h in range(wl.H):
            G = h // g
            s = [sum(float(q[0, r, h, c]) * float(K[0, G, j, c]) for c in range(wl.d)) / math.sqrt(wl.d)
                 for j in range(L - wl.n_q + r + 1)]
            m = max(s)
            den = sum(math.exp(v - m) for v in s)
            ref_lse = m + math.log(den)
            assert lse[0, r, h] == pytest.approx(ref_lse, abs=1e-12)
            for c in range(wl.d):
                num = sum(math.exp(s[j] - ref_lse) * float(V[0, G, j, c]) for j in range(len(s)))
                ab = sum(math.exp(s[j] - ref_lse) * abs(float(V[0, G, j, c])) for j in range(len(s)))
                assert out[0, r, h, c] == pytest.approx(num, abs=1e-12)
                assert absm[0, r, h, c] == pytest.approx(ab, abs=1e-12)


def test_P16d_causal_limit(orc):
    wl, x = _case(B=1, seed=4)
    out, _, _ = orc.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv)
    L = int(x["seq_len"][0])
    r = 2
    lim = L - wl.n_q + r  # last key row r sees
    K2, V2 = x["K"].clone(), x["V"].clone()
    K2[:, :, lim + 1:] = 3.0
    V2[:, :, lim + 1:] = -7.0
    o2, _, _ = orc.question_attention(x["q"], K2, V2, x["seq_len"], wl.vb, wl.nv)
    assert np.array_equal(out[0, :r + 1], o2[0, :r + 1])      # rows 0..r unaffected
    assert not np.allclose(out[0, r + 1], o2[0, r + 1])       # row r + 1 sees key lim + 1
    V3 = x["V"].clone()
    V3[:, :, lim] = 5.0
    o3, _, _ = orc.question_attention(x["q"], x["K"], V3, x["seq_len"], wl.vb, wl.nv)
    assert not np.allclose(out[0, r], o3[0, r])               # key lim is inside row r's range


def test_P16e_constant_v_and_lse_shift(orc):
    wl, x = _case(seed=5)
    Vc = torch.full_like(x["V"], 0.75)
    out, lse, _ = orc.question_attention(x["q"], x["K"], Vc, x["seq_len"], wl.vb, wl.nv)
    assert np.allclose(out, 0.75, atol=1e-13, rtol=0)
    o1, l1, _ = orc.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv)
    o2, l2, _ = orc.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, lse_in=l1 + 0.5)
    assert np.allclose(o2, o1 * math.exp(-0.5), atol=1e-13, rtol=1e-12)
    assert np.array_equal(l2, l1 + 0.5)
