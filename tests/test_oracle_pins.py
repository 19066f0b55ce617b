"""Pins of the fp64 CPU oracle against things other than itself (-m "not gpu").

Each test names its pin and the passage or closed
form it comes from.  Independent references are: values printed in SPEC.md /
PAPER.md (tests/golden/spec_examples.json), closed forms, invariants, and
textbook/library routines (torch float64 softmax / SDPA / logsumexp, numpy
lexsort) on small inputs.  Plausible oracle mistakes (dropped text term,
wrong causal limit, wrong GQA mapping, transposed K/V, missing 1/S or 1/N_f,
wrong tie-break) each fail at least one test here.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from paper_2510_17777_b200 import inputs as gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def bf(x):
    return torch.as_tensor(x, dtype=torch.float64).to(torch.float32).to(torch.bfloat16)


def _ref_relevance(q, K, seq_len, vb, nv, flags, shared=False):
    """Materialized attention with torch.softmax (library) -> visual column
    mass summed over query rows and heads (SPEC.md:374 'oracle that
    materializes full attention probs and column-sums visual columns')."""
    B, n_q, H, d = q.shape
    Hkv = K.shape[1]
    g = H // Hkv
    out = []
    for b in range(B):
        L = int(seq_len[b])
        per_g = []
        for G in range(Hkv):
            qq = q[b, :, G * g:(G + 1) * g, :].to(torch.float64)       # [nq][g][d]
            kk = K[b, G, :L, :].to(torch.float64)                       # [L][d]
            logits = torch.einsum("rhd,jd->rhj", qq, kk) / math.sqrt(d)
            mask = torch.zeros(n_q, 1, L, dtype=torch.bool)
            for r in range(n_q):
                mask[r, 0, L - n_q + r + 1:] = True                     # causal
            if flags & 1:                                               # VISUAL_ONLY
                vis = torch.zeros(L, dtype=torch.bool)
                vis[vb:vb + nv] = True
                mask = mask | ~vis
            logits = logits.masked_fill(mask, float("-inf"))
            P = torch.softmax(logits, dim=-1)
            per_g.append(P[:, :, vb:vb + nv].sum(dim=(0, 1)))
        if shared:
            out.append(torch.stack(per_g).sum(0, keepdim=True))
        else:
            out.append(torch.stack(per_g))
    return torch.stack(out).numpy()


# ----------------------------------------------------------------- generator


def test_splitmix64_reference_stream():
    exp = [int(h, 16) for h in GOLD["splitmix64_seed0"]["outputs_hex"]]
    got = gen.splitmix64(torch.arange(1, 4, dtype=torch.int64) * gen.GOLDEN).tolist()
    assert [x & (2**64 - 1) for x in got] == exp
    for e in range(1, 50):
        z = (e * (gen.GOLDEN & (2**64 - 1)) + 12345) & (2**64 - 1)
        t = gen.splitmix64(torch.tensor([gen._s64(z)], dtype=torch.int64)).item() & (2**64 - 1)
        assert t == gen.splitmix64_py(z)


def test_generator_determinism_and_moments():
    a = gen.normal("x", 3, 200000)
    b = gen.normal("x", 3, 200000)
    c = gen.normal("x", 4, 200000)
    assert torch.equal(a, b) and not torch.equal(a, c)
    assert abs(a.mean().item()) < 0.01 and abs(a.std().item() - 1) < 0.01
    wl = gen.CONFIGS["toy"]
    x1 = gen.make_decode_inputs(wl, seed=1)
    x2 = gen.make_decode_inputs(wl, seed=1)
    for key in ("q", "K", "V", "seq_len"):
        assert torch.equal(x1[key], x2[key])
    assert x1["K"].shape == (1, 2, wl.capacity, 64)


# ----------------------------------------------------------------- P1, P2


def test_P1_spec_worked_example(orc):
    e = GOLD["P1_relevance_worked_example"]
    q = bf(e["q"]).view(1, 1, 1, 1)
    # visual keys [2],[0]; a third row holds the query token itself and is
    # excluded by VISUAL_ONLY ("no other entries").
    K = bf([[2.0], [0.0], [0.0]]).view(1, 1, 3, 1)
    idx, sc, gap = orc.retrieve(q, K, torch.tensor([3]), 0, 2, e["k"], scale=e["scale"],
                                flags=orc.VISUAL_ONLY)
    assert sc[0, 0].tolist() == pytest.approx(e["scores"], abs=1e-15)
    assert idx[0, 0].tolist() == e["idx"]
    assert gap[0, 0] == pytest.approx((e["scores"][0] - e["scores"][1]) / e["scores"][0])


def test_P2_softmax_closed_forms(orc):
    # equal logits -> [0.5, 0.5]
    q = bf([1.0]).view(1, 1, 1, 1)
    K = bf([[0.5], [0.5], [0.0]]).view(1, 1, 3, 1)
    _, sc, gap = orc.retrieve(q, K, torch.tensor([3]), 0, 2, 1, scale=1.0, flags=orc.VISUAL_ONLY)
    assert sc[0, 0].tolist() == pytest.approx([0.5, 0.5], abs=1e-15) and gap[0, 0] == 0.0
    # [[x, 0]] -> [e^x/(e^x+1), 1/(e^x+1)] with x = bf16(ln 2) (SPEC.md:47 closed form)
    x = float(bf(math.log(2.0)))
    K = bf([[x], [0.0], [0.0]]).view(1, 1, 3, 1)
    _, sc, _ = orc.retrieve(q, K, torch.tensor([3]), 0, 2, 1, scale=1.0, flags=orc.VISUAL_ONLY)
    assert sc[0, 0].tolist() == pytest.approx([math.exp(x) / (math.exp(x) + 1),
                                               1 / (math.exp(x) + 1)], abs=1e-15)


# ----------------------------------------------------------------- P3, P7, P10


def test_P3_attention_special_cases(orc):
    # single key -> output == V, lse == logit
    q = bf(torch.randn(1, 2, 8, generator=torch.Generator().manual_seed(0)))
    K = bf(torch.randn(1, 1, 4, 8, generator=torch.Generator().manual_seed(1)))
    V = bf(torch.randn(1, 1, 4, 8, generator=torch.Generator().manual_seed(2)))
    out, lse = orc.dense_attn(q, K, V, torch.tensor([1]))
    assert np.array_equal(out[0, 0], V[0, 0, 0].double().numpy())
    s = (q[0, 1].double() @ K[0, 0, 0].double()).item() / math.sqrt(8)
    assert lse[0, 1] == pytest.approx(s, abs=1e-15)
    # equal logits (q = 0) -> mean of V rows, lse = log(n)
    q0 = torch.zeros(1, 2, 8, dtype=torch.bfloat16)
    out, lse = orc.dense_attn(q0, K, V, torch.tensor([3]))
    assert np.allclose(out[0, 0], V[0, 0, :3].double().mean(0).numpy(), atol=1e-15)
    assert lse[0, 0] == pytest.approx(math.log(3), abs=1e-15)


@pytest.mark.parametrize("B,H,Hkv,d,L", [(2, 4, 2, 16, 37), (1, 7, 1, 32, 50), (3, 6, 6, 8, 9)])
def test_P7_dense_matches_torch_sdpa(orc, B, H, Hkv, d, L):
    g = torch.Generator().manual_seed(B * 100 + H)
    q = bf(2 * torch.randn(B, H, d, generator=g))
    K = bf(torch.randn(B, Hkv, L + 3, d, generator=g))
    V = bf(torch.randn(B, Hkv, L + 3, d, generator=g))
    seq = torch.tensor([L - b for b in range(B)], dtype=torch.int32)
    out, lse = orc.dense_attn(q, K, V, seq)
    rep = H // Hkv
    for b in range(B):
        Lb = int(seq[b])
        kk = K[b, :, :Lb].double().repeat_interleave(rep, 0)       # [H][L][d]
        vv = V[b, :, :Lb].double().repeat_interleave(rep, 0)
        qq = q[b].double()[:, None, :]                              # [H][1][d]
        ref = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv)[:, 0]
        assert np.allclose(out[b], ref.numpy(), atol=1e-12, rtol=0)
        ref_lse = torch.logsumexp((qq @ kk.transpose(1, 2))[:, 0] / math.sqrt(d), -1)
        assert np.allclose(lse[b], ref_lse.numpy(), atol=1e-12, rtol=0)


def test_P7_full_selection_equals_dense_bitwise(orc):
    wl = gen.DecodeWorkload("p7", 2, 4, 2, 16, 5, 40, 7, 40, 1, 8)
    x = gen.make_decode_inputs(wl, seed=3)
    idx = np.tile(np.arange(wl.nv, dtype=np.int32), (wl.B, wl.Hkv, 1))
    o1, l1 = orc.sparse_decode(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx)
    o2, l2 = orc.dense_attn(x["q_dec"], x["K"], x["V"], x["seq_len"])
    assert np.array_equal(o1, o2) and np.array_equal(l1, l2)


def test_P10_lse_merge_of_a_partition_equals_whole(orc):
    """Closed-form rescaling identity (north star step 3):
    out = sum_i e^{lse_i - M} o_i / sum_i e^{lse_i - M}."""
    wl = gen.DecodeWorkload("p10", 1, 6, 2, 32, 0, 96, 0, 96, 1, 16, sinks=0, needles=0)
    wl.t_after = 1                      # seq = 97 rows; last row is "text"
    x = gen.make_decode_inputs(wl, seed=5)
    rng = np.random.default_rng(0)
    perm = rng.permutation(96)
    A, Bs = np.sort(perm[:40]), np.sort(perm[40:])
    # pieces: A (+ the text row), B, and the text row alone counted once
    oA, lA = orc.sparse_decode(x["q_dec"], x["K"], x["V"], x["seq_len"], 0, 96,
                               np.tile(A.astype(np.int32), (1, 2, 1)))
    seq_vis = torch.tensor([96], dtype=torch.int32)     # drop the text row
    oB, lB = orc.sparse_decode(x["q_dec"], x["K"], x["V"], seq_vis, 0, 96,
                               np.tile(Bs.astype(np.int32), (1, 2, 1)))
    o, l = orc.dense_attn(x["q_dec"], x["K"], x["V"], x["seq_len"])
    M = np.maximum(lA, lB)
    wA, wB = np.exp(lA - M), np.exp(lB - M)
    om = (wA[..., None] * oA + wB[..., None] * oB) / (wA + wB)[..., None]
    assert np.allclose(om, o, atol=1e-12, rtol=0)
    assert np.allclose(M + np.log(wA + wB), l, atol=1e-12, rtol=0)


# ----------------------------------------------------------------- P4, P5


def test_P4_keep_budget(orc):
    for n, s, k in GOLD["P4_keep_budget"]["cases"]:
        assert orc.keep_budget(n, s) == k
    assert orc.keep_budget(5, 1.0) == -1 and orc.keep_budget(5, -0.1) == -1


def test_P5_topk_tie_and_bruteforce(orc):
    e = GOLD["P5_topk_tie"]
    sal = np.array([e["scores"]], np.float32)
    kept, tot = orc.prune(sal, 1 - e["k"] / 3 + 1e-9)     # keep_budget(3, s) == 1
    assert tot == 1 and kept[0].tolist() == e["idx"]
    kept, tot = orc.prune(sal, 0.0)
    assert kept[0].tolist() == [0, 1, 2]
    # 1000 random scores, k=137 vs a full sort by numpy.lexsort
    rng = np.random.default_rng(7)
    v = np.round(rng.random(1000) * 300).astype(np.float32) / 300   # many ties
    s = 1 - 137 / 1000
    assert orc.keep_budget(1000, s) == 137
    kept, tot = orc.prune(v[None], s)
    order = np.lexsort((np.arange(1000), -v.astype(np.float64)))
    assert tot == 137 and kept[0].tolist() == sorted(order[:137].tolist())


def test_P5_prune_per_frame_bruteforce(orc):
    rng = np.random.default_rng(11)
    B, N = 3, 700
    offs = np.array([0, 100, 101, 101, 356, 700], np.int32)    # ragged + empty frame
    sal = (np.round(rng.random((B, N)) * 50) / 50).astype(np.float32)
    s = 0.75
    kept, tot = orc.prune(sal, s, offs)
    assert tot == sum(orc.keep_budget(int(offs[i + 1] - offs[i]), s) for i in range(5))
    for b in range(B):
        ref = []
        for f in range(5):
            a, z = offs[f], offs[f + 1]
            kf = orc.keep_budget(int(z - a), s)
            v = sal[b, a:z].astype(np.float64)
            order = np.lexsort((np.arange(z - a), -v))
            ref += sorted((a + order[:kf]).tolist())
        assert kept[b].tolist() == ref
        assert all(x < y for x, y in zip(ref, ref[1:]))


# ----------------------------------------------------------------- retrieve


@pytest.mark.parametrize("flags", [0, 1])
@pytest.mark.parametrize("n_q,H,Hkv", [(1, 4, 2), (3, 6, 2), (2, 3, 3)])
def test_retrieve_scores_match_materialized_softmax(orc, flags, n_q, H, Hkv):
    wl = gen.DecodeWorkload("rs", 2, H, Hkv, 16, 4, 50, 9, 10, n_q, 16)
    wl.seq_lens = [wl.seq_len, wl.seq_len - 3]
    x = gen.make_decode_inputs(wl, seed=n_q)
    idx, sc, gap = orc.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, flags=flags)
    ref = _ref_relevance(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, flags)
    assert np.allclose(sc, ref, atol=1e-13, rtol=1e-12)
    g = H // Hkv
    tot = sc.sum(-1)
    if flags & 1:       # closed form: the visual shares sum to n_q*g exactly
        assert np.allclose(tot, n_q * g, atol=1e-12)
    else:               # the text rows take a strictly positive share
        assert np.all(tot < n_q * g)
    # selection = first k of a lexsort of the library-computed scores
    for b in range(2):
        for G in range(Hkv):
            order = np.lexsort((np.arange(wl.nv), -ref[b, G]))
            if gap[b, G] > 1e-9:
                assert idx[b, G].tolist() == sorted(order[:wl.k].tolist())


def test_retrieve_shared_sums_groups(orc):
    wl = gen.DecodeWorkload("sh", 1, 6, 3, 16, 4, 60, 5, 12, 1, 16)
    x = gen.make_decode_inputs(wl, seed=2)
    idx, sc, gap = orc.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, flags=orc.SHARED)
    ref = _ref_relevance(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, 0, shared=True)
    assert sc.shape == (1, 1, 60) and np.allclose(sc, ref, atol=1e-13, rtol=1e-12)


def test_retrieve_lse_in_equals_full_prefix(orc):
    wl = gen.DecodeWorkload("lse", 1, 4, 2, 16, 4, 40, 6, 8, 2, 16)
    x = gen.make_decode_inputs(wl, seed=9)
    q, K = x["q"].double(), x["K"].double()
    L = int(x["seq_len"][0])
    lse = torch.zeros(1, 2, 4, dtype=torch.float64)
    for r in range(2):
        for h in range(4):
            s = K[0, h // 2, :L - 2 + r + 1] @ q[0, r, h] / 4.0
            lse[0, r, h] = torch.logsumexp(s, 0)
    _, s1, _ = orc.retrieve(x["q"], x["K"], x["seq_len"], 4, 40, 8)
    _, s2, _ = orc.retrieve(x["q"], x["K"], x["seq_len"], 4, 40, 8, lse_in=lse.numpy())
    assert np.allclose(s1, s2, atol=1e-14, rtol=1e-12)


def test_P11_single_head_selection_is_raw_dot_topk(orc):
    """n_q=1, g=1: exp is monotone so the set is top-k of raw q.K (GEMV +
    sort), for either normalisation."""
    wl = gen.DecodeWorkload("p11", 1, 2, 2, 32, 3, 300, 5, 30, 1, 64)
    x = gen.make_decode_inputs(wl, seed=4)
    for flags in (0, 1):
        idx, _, _ = orc.retrieve(x["q"], x["K"], x["seq_len"], 3, 300, 30, flags=flags)
        for G in range(2):
            dots = (x["K"][0, G, 3:303].double() @ x["q"][0, 0, G].double())
            top = torch.topk(dots, 30).indices.sort().values.tolist()
            assert idx[0, G].tolist() == top


def test_P6_permutation_equivariance(orc):
    wl = gen.DecodeWorkload("p6", 1, 4, 2, 16, 2, 64, 3, 16, 1, 64)
    x = gen.make_decode_inputs(wl, seed=6)
    idx, sc, _ = orc.retrieve(x["q"], x["K"], x["seq_len"], 2, 64, 16)
    perm = torch.from_numpy(np.random.default_rng(1).permutation(64))
    K2 = x["K"].clone()
    K2[:, :, 2:66] = x["K"][:, :, 2 + perm]
    idx2, sc2, _ = orc.retrieve(x["q"], K2, x["seq_len"], 2, 64, 16)
    assert np.allclose(sc2, sc[:, :, perm.numpy()], atol=1e-15, rtol=1e-13)
    inv = torch.argsort(perm).numpy()
    for G in range(2):
        assert sorted(inv[idx[0, G]].tolist()) == idx2[0, G].tolist()
    # output unchanged when the same rows are attended (permuted storage)
    o1, _ = orc.sparse_decode(x["q_dec"], x["K"], x["V"], x["seq_len"], 2, 64, idx)
    V2 = x["V"].clone()
    V2[:, :, 2:66] = x["V"][:, :, 2 + perm]
    o2, _ = orc.sparse_decode(x["q_dec"], K2, V2, x["seq_len"], 2, 64, idx2)
    assert np.allclose(o1, o2, atol=1e-12)


def test_P6_shift_invariance_single_head(orc):
    """Adding c*q/|q|^2-ish offsets to every visual key shifts all visual
    logits by the same constant; with VISUAL_ONLY the scores are unchanged."""
    d = 8
    q = bf([[1.0] + [0.0] * (d - 1)]).view(1, 1, 1, d)
    K = bf(torch.randn(1, 1, 41, d, generator=torch.Generator().manual_seed(3)))
    _, s1, _ = orc.retrieve(q, K, torch.tensor([41]), 0, 40, 5, flags=orc.VISUAL_ONLY)
    K2 = K.clone()
    K2[0, 0, :40, 0] = bf(K[0, 0, :40, 0].double() + 2.0)
    if torch.equal(K2[0, 0, :40, 0].double() - K[0, 0, :40, 0].double(),
                   torch.full((40,), 2.0, dtype=torch.float64)):
        _, s2, _ = orc.retrieve(q, K2, torch.tensor([41]), 0, 40, 5, flags=orc.VISUAL_ONLY)
        assert np.allclose(s1, s2, atol=1e-15, rtol=1e-12)


def test_P13_duplicates_tie_to_lower_index(orc):
    wl = gen.DecodeWorkload("p13", 1, 2, 1, 16, 2, 50, 3, 10, 1, 64, sinks=0, needles=0)
    x = gen.make_decode_inputs(wl, seed=8)
    idx, sc, _ = orc.retrieve(x["q"], x["K"], x["seq_len"], 2, 50, 10)
    order = np.lexsort((np.arange(50), -sc[0, 0]))
    kth = int(order[9])                           # the k-th best row
    for dup in (max(kth - 1, 0) if kth > 0 else None, min(kth + 1, 49)):
        if dup is None or dup in order[:10].tolist():
            continue
        K2 = x["K"].clone()
        K2[0, 0, 2 + dup] = K2[0, 0, 2 + kth]
        idx2, sc2, gap2 = orc.retrieve(x["q"], K2, x["seq_len"], 2, 50, 10)
        assert sc2[0, 0, dup] == sc2[0, 0, kth] and gap2[0, 0] == 0.0
        want = min(dup, kth)
        lose = max(dup, kth)
        assert want in idx2[0, 0].tolist() and lose not in idx2[0, 0].tolist()


def test_P9_planted_needles_and_gqa_mapping(orc):
    """A visual key along group G's mean query direction is retrieved for
    group G at decode sparsity 0.90, and NOT
    for the other group (pins kv = h // g, reading A5)."""
    wl = gen.DecodeWorkload("p9", 2, 8, 2, 64, 8, 640, 20, 64, 1, 64, sinks=8, needles=0)
    x = gen.make_decode_inputs(wl, seed=12)
    K = x["K"].clone()
    q = x["q"].double()
    needles = {0: [33, 200, 333, 480, 601], 1: [70, 150, 260, 390, 555]}
    for b in range(2):
        for G in range(2):
            u = q[b, 0, G * 4:(G + 1) * 4].sum(0)
            u = u / u.norm()
            for j in needles[G]:
                K[b, G, 8 + j] = bf(6.0 * u)
    assert orc.keep_budget(640, 0.9) == 64
    idx, _, _ = orc.retrieve(x["q"], K, x["seq_len"], 8, 640, 64)
    for b in range(2):
        for G in range(2):
            got = set(idx[b, G].tolist())
            assert set(needles[G]) <= got


# ----------------------------------------------------------------- salience P8


def test_P8_salience_uniform_and_readoff(orc):
    Q = torch.zeros(1, 4, 2, 8, dtype=torch.bfloat16)
    K = bf(torch.randn(1, 4, 2, 8, generator=torch.Generator().manual_seed(0)))
    sal = orc.salience(Q, K, 0, orc.SAL_INTRA_VISUAL)
    assert np.allclose(sal, 0.25, atol=1e-15)
    # SUMMARY, N=2, d=1: P[0,:] = softmax([a0, a1, a2]) closed form
    Q = bf([[[1.0]], [[0.0]], [[0.0]]]).view(1, 3, 1, 1)
    K = bf([[[-3.0]], [[2.0]], [[0.0]]]).view(1, 3, 1, 1)
    sal = orc.salience(Q, K, 1, orc.SAL_SUMMARY, scale=1.0)
    z = math.exp(-3) + math.exp(2) + 1
    assert sal[0].tolist() == pytest.approx([math.exp(2) / z, 1 / z], abs=1e-15)


@pytest.mark.parametrize("S,mode", [(0, 2), (1, 0), (3, 1)])
def test_P8_salience_matches_materialized_softmax(orc, S, mode):
    wl = gen.PrefillWorkload("p8", 2, S, 37, 3, 16)
    x = gen.make_prefill_inputs(wl, seed=S)
    sal = orc.salience(x["Qe"], x["Ke"], S, mode)
    Q, K = x["Qe"].double(), x["Ke"].double()
    P = torch.softmax(torch.einsum("fihc,fjhc->fhij", Q, K) / 4.0, -1)    # [F][He][T][T]
    if mode == 2:
        ref = P[:, :, :, :].mean(2).mean(1)                               # mean over rows i
    else:
        ref = P[:, :, :S, S:].mean(2).mean(1)
    assert np.allclose(sal, ref.numpy(), atol=1e-15, rtol=1e-12)
    if mode == 2:
        assert np.allclose(sal.sum(-1), 1.0, atol=1e-12)


def test_P8_salience_permutation_equivariant(orc):
    wl = gen.PrefillWorkload("p8p", 1, 0, 40, 2, 8)
    x = gen.make_prefill_inputs(wl, seed=1)
    perm = torch.from_numpy(np.random.default_rng(2).permutation(40))
    s1 = orc.salience(x["Qe"], x["Ke"], 0, 2)
    s2 = orc.salience(x["Qe"][:, perm], x["Ke"][:, perm], 0, 2)
    assert np.allclose(s2[0], s1[0, perm.numpy()], atol=1e-15, rtol=1e-12)


def test_salience_mode_mismatch_is_error(orc):
    x = gen.make_prefill_inputs(gen.PrefillWorkload("e", 1, 1, 8, 1, 8), seed=0)
    with pytest.raises(orc.OracleError):
        orc.salience(x["Qe"], x["Ke"], 1, orc.SAL_INTRA_VISUAL)


def test_retrieve_bad_args(orc):
    x = gen.make_decode_inputs(gen.CONFIGS["toy"], seed=0)
    with pytest.raises(orc.OracleError):
        orc.retrieve(x["q"], x["K"], x["seq_len"], 8, 512, 513)


def test_oracle_thread_count_bitwise(orc):
    wl = gen.DecodeWorkload("thr", 2, 4, 2, 32, 4, 128, 8, 16, 1, 32)
    x = gen.make_decode_inputs(wl, seed=1)
    a = orc.retrieve(x["q"], x["K"], x["seq_len"], 4, 128, 16, nthreads=1)
    b = orc.retrieve(x["q"], x["K"], x["seq_len"], 4, 128, 16, nthreads=4)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


# ---------------------------------------------------------------- f4(i) RoPE remap pins
def _rope_inputs(B, Hkv, cap, d, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16)


def test_rope_remap_spec_example_plan(orc):
    """visual span 10..20, kept {12, 15, 19} -> new {10, 11, 12}, text 21 -> 13."""
    K = _rope_inputs(1, 1, 40, 8, 0)
    _, rows = orc.rope_remap(K, [30], 10, 11, [[2, 5, 9]], 10000.0)
    assert list(rows[0][:13]) == list(range(10)) + [12, 15, 19]
    assert rows[0][13] == 21                      # the text start moved from 21 to 13
    assert list(rows[0][13:22]) == list(range(21, 30)) and rows[0][22] == -1


def test_rope_remap_matches_complex_rotation(orc):
    """Rotate-half RoPE == multiplying (x[c] + i x[c + d/2]) by e^{i p base^(-2c/d)}
    (a different formulation, Python complex arithmetic)."""
    import cmath
    d, base = 16, 10000.0
    K = _rope_inputs(1, 2, 24, d, 1)
    out, rows = orc.rope_remap(K, [24], 4, 10, [[0, 3, 7, 9]], base)
    Kd = K.double().numpy()
    for G in range(2):
        for w in range(18):
            old = rows[0][w]
            for c in range(d // 2):
                z = complex(Kd[0, G, old, c], Kd[0, G, old, c + d // 2]) * cmath.exp(1j * w * base ** (-2 * c / d))
                assert abs(out[0, G, w, c] - z.real) < 1e-12 and abs(out[0, G, w, c + d // 2] - z.imag) < 1e-12


def test_rope_remap_relative_position_and_norm(orc):
    """RoPE's defining property: a rotated query-key dot product depends only on the
    position difference; rotations preserve the norm; position 0 is the identity."""
    d = 64
    K = _rope_inputs(1, 1, 40, d, 2)
    for a, b_ in ((1, 5), (2, 9)):             # put the same (q, k) pair at rows (a, a+1) and (b, b+1)
        K[0, 0, b_] = K[0, 0, a]
        K[0, 0, b_ + 1] = K[0, 0, a + 1]
    out, _ = orc.rope_remap(K, [30], 12, 8, [[1, 4]], 500000.0)
    x = K.double().numpy()[0, 0]
    assert np.array_equal(out[0, 0, 0], x[0])                                   # p = 0
    for w in range(12):
        assert abs(np.linalg.norm(out[0, 0, w]) - np.linalg.norm(x[w])) < 1e-9 * np.linalg.norm(x[w])
    assert abs(out[0, 0, 1] @ out[0, 0, 2] - out[0, 0, 5] @ out[0, 0, 6]) < 1e-9
    assert abs(out[0, 0, 2] @ out[0, 0, 3] - out[0, 0, 9] @ out[0, 0, 10]) < 1e-9


# ---------------------------------------------------------------- page summaries (f2(ii))

def _pages_case(B=2, H=6, Hkv=2, d=16, vb=3, nv=48, n_q=1, seed=0):
    g = torch.Generator().manual_seed(seed)
    cap = vb + nv + 5
    q = (torch.randn(B, n_q, H, d, generator=g) * 2).to(torch.bfloat16)
    K = torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16)
    return q, K, vb, nv


def test_p14_page_retrieval_worked_example(orc):
    """PAPER.md:527 (Quest) / reading A22: the hand-worked two-page case."""
    ex = GOLD["P14_page_retrieval"]
    K = torch.tensor(ex["K_visual"], dtype=torch.float32).view(1, 1, 4, 1).to(torch.bfloat16)
    kmax, kmin = orc.page_summary(K, 0, 4, ex["page"])
    assert kmax.ravel().tolist() == [2.0, 3.0] and kmin.ravel().tolist() == [0.0, -1.0]
    for case in ex["cases"]:
        q = torch.tensor(case["q"], dtype=torch.float32).view(1, 1, 1, 1).to(torch.bfloat16)
        idx, sc, _ = orc.retrieve_pages(q, kmax, kmin, case["k_pages"], scale=ex["scale"])
        assert np.allclose(sc.ravel(), case["scores"], rtol=1e-14, atol=0)
        assert idx.ravel().tolist() == case["page_idx"]


def test_page_summary_is_elementwise_max_min(orc):
    """The summary is the per-page elementwise max / min (a library reduction)."""
    q, K, vb, nv = _pages_case()
    for page in (1, 4, 16):
        kmax, kmin = orc.page_summary(K, vb, nv, page)
        vis = K[:, :, vb:vb + nv].float().numpy().astype(np.float64)
        B, Hkv, _, d = vis.shape
        r = vis.reshape(B, Hkv, nv // page, page, d)
        assert np.array_equal(kmax, r.max(axis=3)) and np.array_equal(kmin, r.min(axis=3))


@pytest.mark.parametrize("n_q,H,Hkv", [(1, 6, 2), (2, 3, 3), (1, 4, 1)])
def test_page_one_equals_visual_only_retrieve(orc, n_q, H, Hkv):
    """page = 1: the bound is the logit itself and the softmax over pages is the softmax
    over the visual rows -> o_retrieve with VISUAL_ONLY, scores and indices."""
    q, K, vb, nv = _pages_case(H=H, Hkv=Hkv, n_q=n_q, seed=3 + n_q)
    seq = torch.full((q.shape[0],), vb + nv + 5, dtype=torch.int32)
    kmax, kmin = orc.page_summary(K, vb, nv, 1)
    pi, ps, _ = orc.retrieve_pages(q, kmax, kmin, 7)
    ri, rs, _ = orc.retrieve(q, K, seq, vb, nv, 7, flags=orc.VISUAL_ONLY)
    assert np.allclose(ps, rs, rtol=1e-12, atol=0)
    assert np.array_equal(pi, ri)


def test_page_bound_dominates_every_row_logit(orc):
    """Quest's bound: scale*sum_c max(q kmax, q kmin) >= scale * q.K_j for every row j of
    the page, with equality when the page's rows are identical (exact logits by torch)."""
    q, K, vb, nv = _pages_case(B=1, H=2, Hkv=1, d=32, nv=64, seed=9)
    page = 8
    K[0, 0, vb + 16:vb + 24] = K[0, 0, vb + 16]  # page 2: identical rows
    kmax, kmin = orc.page_summary(K, vb, nv, page)
    scale = 0.25
    # one head at a time, single page kept per call: the score of a 1-page set is 1, so
    # read the bound from two pages: score_p / score_0 = exp(ub_p - ub_0)
    vis = K[0, 0, vb:vb + nv].double()
    for h in range(2):
        qh = q[:, :, h:h + 1]
        _, sc, _ = orc.retrieve_pages(qh, kmax[:, :1], kmin[:, :1], 1, scale=scale)
        ub_rel = np.log(sc[0, 0]) - np.log(sc[0, 0, 0])  # ub_p - ub_0
        logits = scale * (vis @ q[0, 0, h].double()).numpy()
        mx = logits.reshape(nv // page, page).max(axis=1)
        # ub_p - ub_0 >= ... : compare both sides against page 2 (tight) to remove ub_0
        tight = mx[2]
        ub_p = ub_rel - ub_rel[2] + tight
        assert np.all(ub_p >= mx - 1e-9)
        assert abs(ub_p[2] - mx[2]) < 1e-9


def test_page_retrieval_permutation_equivariant(orc):
    q, K, vb, nv = _pages_case(B=1, seed=11)
    page = 4
    kmax, kmin = orc.page_summary(K, vb, nv, page)
    perm = np.random.default_rng(1).permutation(nv // page)
    _, s0, _ = orc.retrieve_pages(q, kmax, kmin, 3)
    _, s1, _ = orc.retrieve_pages(q, kmax[:, :, perm], kmin[:, :, perm], 3)
    assert np.allclose(s1, s0[:, :, perm], rtol=1e-12, atol=0)


# ---------------------------------------------------------------- mRoPE remap (f4(i))

def _grid_coords(T, Hh, Ww):
    t, h, w = np.meshgrid(np.arange(T), np.arange(Hh), np.arange(Ww), indexing="ij")
    return np.stack([t.ravel(), h.ravel(), w.ravel()], axis=-1).astype(np.int32)


def test_p15_mrope_plan_spec_example(orc):
    ex = GOLD["P15_mrope_plan"]
    coords = np.array(ex["kept_coords"], np.int32)[None]
    nc, ts = orc.mrope_plan(coords, ex["vb"], np.arange(4, dtype=np.int32)[None])
    assert nc[0].tolist() == ex["new_coords"] and int(ts[0]) == ex["text_start"]


def test_mrope_plan_full_grid_is_identity(orc):
    coords = _grid_coords(3, 4, 5)[None]
    n = coords.shape[1]
    nc, ts = orc.mrope_plan(coords, 7, np.arange(n, dtype=np.int32)[None])
    assert np.array_equal(nc, coords) and int(ts[0]) == 7 + 1 + 4


def test_mrope_plan_rank_compression_injective_idempotent(orc):
    """Per dimension the plan is numpy's unique-inverse (coordinate compression); distinct
    triples stay distinct over random prunings; re-planning is the identity;
    the text start exceeds every remapped position."""
    rng = np.random.default_rng(0)
    coords = _grid_coords(6, 5, 7)[None]
    n = coords.shape[1]
    for _ in range(200):
        k = int(rng.integers(1, n))
        kept = np.sort(rng.choice(n, k, replace=False)).astype(np.int32)[None]
        nc, ts = orc.mrope_plan(coords, 3, kept)
        kc = coords[0, kept[0]]
        for x in range(3):
            _, inv = np.unique(kc[:, x], return_inverse=True)
            assert np.array_equal(nc[0, :, x], inv)
        assert len({tuple(r) for r in nc[0]}) == k
        nc2, ts2 = orc.mrope_plan(nc, 3, np.arange(k, dtype=np.int32)[None])
        assert np.array_equal(nc2, nc) and ts2[0] == ts[0]
        assert ts[0] > 3 + nc.max()


def test_mrope_plan_rejects_duplicate_triples(orc):
    coords = np.array([[[0, 0, 0], [0, 0, 0], [1, 0, 0]]], np.int32)
    with pytest.raises(orc.OracleError):
        orc.mrope_plan(coords, 0, np.array([[0, 1]], np.int32))


def test_mrope_diagonal_coords_equal_unified_rope(orc):
    """Kept tokens on the diagonal (i, i, i): every section sees position vb + rank, the
    text start is vb + k -- exactly the unified remap (o_rope_remap), bitwise in fp64."""
    g = torch.Generator().manual_seed(4)
    B, Hkv, d, vb, nv, ta = 1, 2, 16, 3, 20, 4
    cap = vb + nv + ta
    K = torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16)
    seq = np.array([cap], np.int32)
    coords = np.stack([np.arange(nv)] * 3, axis=-1).astype(np.int32)[None]
    kept = np.array([[1, 4, 5, 9, 15, 19]], np.int32)
    nc, ts = orc.mrope_plan(coords, vb, kept)
    a, ra = orc.mrope_remap(K, seq, vb, nv, kept, nc, ts, [2, 3, 3], 10000.0)
    b, rb = orc.rope_remap(K, seq, vb, nv, kept, 10000.0)
    assert np.array_equal(ra, rb) and np.array_equal(a, b)


def test_mrope_relative_position_property(orc):
    """Shifting every position by a common constant (here: 4 more system rows) leaves the
    dot products between re-rotated kept visual keys unchanged (RoPE's relative-position
    property per section, 1e-9)."""
    g = torch.Generator().manual_seed(6)
    Hkv, d, nv, ta = 1, 24, 30, 2
    coords = _grid_coords(2, 3, 5)[None]
    kept = np.array([[0, 3, 7, 8, 14, 22, 29]], np.int32)
    outs = []
    for vb in (2, 6):
        cap = vb + nv + ta
        Kfull = torch.randn(1, Hkv, 6 + nv + ta, d, generator=torch.Generator().manual_seed(6)).to(torch.bfloat16)
        K = torch.cat([Kfull[:, :, :vb], Kfull[:, :, 6:]], dim=2)  # same visual / text keys, vb system rows
        nc, ts = orc.mrope_plan(coords, vb, kept)
        o, _ = orc.mrope_remap(K, np.array([cap], np.int32), vb, nv, kept, nc, ts, [4, 4, 4], 10000.0)
        vis = o[0, 0, vb:vb + kept.shape[1]]
        outs.append(vis @ vis.T)
    assert np.allclose(outs[0], outs[1], rtol=0, atol=1e-9)
