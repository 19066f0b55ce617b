"""GPU parity tests (-m gpu): the CUDA path through the C ABI vs the fp64 CPU
oracle on identical seeded inputs (SURVEY.md 8(c) c6 rules, tests/parity.py).

Sizes: small cases spanning several tiles with ragged tails; the BASELINE
configs at full size (long-video, multi-turn, nvila-4k; the sweep on sampled
batch rows) in the launch configuration bench.py times; edge cases (k=0,
k=N_v, duplicates, ragged seq_len, n_q>1, lse_in, SHARED, bad indices).
"""
import math
import os

import numpy as np
import pytest
import torch

from paper_2510_17777_b200 import inputs as gen
from tests import parity

pytestmark = pytest.mark.gpu

NTH = os.cpu_count() or 1


@pytest.fixture(scope="module")
def svl():
    from paper_2510_17777_b200 import build, svl as mod
    build.build()
    mod.lib()
    return mod


def _gen(wl, seed, big=False):
    x = gen.make_decode_inputs(wl, seed=seed, device="cuda" if big else "cpu")
    cpu = {k: v.cpu() for k, v in x.items()}
    dev = {k: v.cuda() for k, v in x.items()}
    return cpu, dev


def _retrieve_both(svl, orc, wl, cpu, dev, flags=0, lse=None, k=None):
    k = wl.k if k is None else k
    U = 1 if flags & svl.SVL_SELECT_SHARED else wl.Hkv
    sc = torch.empty(wl.B, U, wl.nv, dtype=torch.float32, device="cuda")
    lse_dev = None if lse is None else torch.as_tensor(lse, dtype=torch.float32).cuda()
    idx = svl.retrieve(dev["q"], dev["K"], dev["seq_len"], wl.vb, wl.nv, k, flags=flags,
                       lse_in=lse_dev, scores_out=sc)
    torch.cuda.synchronize()
    oi, osc, gap = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, k, flags=flags,
                                lse_in=lse, nthreads=NTH)
    return idx.cpu().numpy(), sc.cpu().numpy(), oi, osc, gap


def _check_scores(sc, osc):
    err = np.abs(sc - osc) / np.maximum(np.abs(osc), 1e-30)
    big = osc > osc.max() * 1e-6          # relative error on non-negligible scores
    assert err[big].max() < 2e-5, err[big].max()


@pytest.mark.parametrize("name", ["toy", "nvila-4k", "long-video"])
@pytest.mark.parametrize("flags", [0, 1])
def test_retrieve_configs(svl, orc, name, flags):
    wl = gen.CONFIGS[name]
    cpu, dev = _gen(wl, seed=1, big=(name != "toy"))
    idx, sc, oi, osc, gap = _retrieve_both(svl, orc, wl, cpu, dev, flags)
    _check_scores(sc, osc)
    frac = parity.check_indices(idx, osc, gap, wl.k)
    print(f"{name} flags={flags}: strict-regime fraction {frac:.2f}")


@pytest.mark.parametrize("name", ["toy", "nvila-4k", "long-video"])
def test_retrieve_gapped_strict_bitexact(svl, orc, name):
    base = gen.CONFIGS[name]
    # gapped variant: raise gamma until every unit's
    # oracle rel_gap >= 1e-3, so the strict bit-exact regime covers all units
    for gamma in (4.0, 8.0, 16.0):
        wl = gen.DecodeWorkload(**{**base.__dict__, "gap_gamma": gamma, "sinks": 0, "needles": 0})
        cpu, dev = _gen(wl, seed=2, big=(name != "toy"))
        idx, sc, oi, osc, gap = _retrieve_both(svl, orc, wl, cpu, dev)
        if gap.min() > 1e-3:
            break
    assert gap.min() > 1e-3, gap.min()
    assert parity.check_indices(idx, osc, gap, wl.k) == 1.0
    assert np.array_equal(idx, oi)


def test_retrieve_multi_turn_full(svl, orc):
    wl = gen.CONFIGS["multi-turn"]
    cpu, dev = _gen(wl, seed=3, big=True)
    idx, sc, oi, osc, gap = _retrieve_both(svl, orc, wl, cpu, dev)
    _check_scores(sc, osc)
    parity.check_indices(idx, osc, gap, wl.k)


@pytest.mark.parametrize("n_q,H,Hkv,d", [(1, 8, 8, 64), (4, 28, 4, 128), (2, 16, 2, 128), (3, 6, 2, 64)])
def test_retrieve_shapes_ragged(svl, orc, n_q, H, Hkv, d):
    wl = gen.DecodeWorkload("rg", 3, H, Hkv, d, 13, 1237, 41, 123, n_q, 100)
    wl.seq_lens = [wl.seq_len, wl.seq_len - 17, wl.seq_len - 40 + n_q]
    cpu, dev = _gen(wl, seed=n_q)
    for flags in (0, 1, 2):
        idx, sc, oi, osc, gap = _retrieve_both(svl, orc, wl, cpu, dev, flags)
        _check_scores(sc, osc)
        parity.check_indices(idx, osc, gap, wl.k)


def test_retrieve_lse_in(svl, orc):
    wl = gen.DecodeWorkload("lse", 2, 28, 4, 128, 32, 3000, 100, 300, 2, 256)
    cpu, dev = _gen(wl, seed=5)
    # the full-prefix LSE computed independently with torch float64
    q, K = cpu["q"].double(), cpu["K"].double()
    L = wl.seq_len
    lse = torch.zeros(2, 2, 28, dtype=torch.float64)
    for b in range(2):
        for r in range(2):
            for h in range(28):
                s = K[b, h // 7, :L - 2 + r + 1] @ q[b, r, h] / math.sqrt(128)
                lse[b, r, h] = torch.logsumexp(s, 0)
    idx, sc, oi, osc, gap = _retrieve_both(svl, orc, wl, cpu, dev, lse=lse.numpy())
    _check_scores(sc, osc)
    parity.check_indices(idx, osc, gap, wl.k)


@pytest.mark.parametrize("k", [0, 1, 1237])
def test_retrieve_k_edges(svl, orc, k):
    wl = gen.DecodeWorkload("ke", 1, 4, 2, 64, 3, 1237, 9, k, 1, 100)
    cpu, dev = _gen(wl, seed=7)
    idx, sc, oi, osc, gap = _retrieve_both(svl, orc, wl, cpu, dev, k=k)
    assert np.array_equal(idx, oi)


def test_retrieve_duplicates_tie_to_lower_index(svl, orc):
    wl = gen.DecodeWorkload("dup", 1, 14, 2, 128, 8, 4000, 20, 400, 1, 256)
    cpu, dev = _gen(wl, seed=8)
    _, _, oi, osc, _ = _retrieve_both(svl, orc, wl, cpu, dev)
    for G in range(2):
        order = np.lexsort((np.arange(wl.nv), -osc[0, G]))
        kth = int(order[wl.k - 1])
        # duplicate the k-th row into unselected rows before and after it
        for dup in [j for j in order[wl.k:wl.k + 50].tolist()][:6]:
            cpu["K"][0, G, wl.vb + dup] = cpu["K"][0, G, wl.vb + kth]
    dev["K"] = cpu["K"].cuda()
    idx, sc, oi, osc, gap = _retrieve_both(svl, orc, wl, cpu, dev)
    assert np.array_equal(idx, oi)                     # exact, even at gap 0
    for G in range(2):
        s = sc[0, G]
        vals, counts = np.unique(s[idx[0, G]], return_counts=True)
        assert counts.max() >= 1


def test_retrieve_deterministic_bitwise(svl):
    wl = gen.CONFIGS["nvila-4k"]
    x = gen.make_decode_inputs(wl, seed=9, device="cuda")
    outs = []
    for _ in range(3):
        sc = torch.empty(1, 4, wl.nv, device="cuda")
        idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, scores_out=sc)
        outs.append((idx.clone(), sc.clone()))
    for i, s in outs[1:]:
        assert torch.equal(i, outs[0][0]) and torch.equal(s, outs[0][1])


def test_retrieve_planted_needles(svl):
    wl = gen.DecodeWorkload("niah", 2, 28, 4, 128, 32, 256 * 64, 64, 0, 1, 256, sinks=8,
                            needles=5)
    wl.k = svl.keep_budget(wl.nv, 0.90)
    x = gen.make_decode_inputs(wl, seed=10, device="cuda")
    idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k).cpu().numpy()
    depth = [int((2 * i + 1) * wl.nv / 10) for i in range(5)]
    for b in range(2):
        for G in range(4):
            assert set(depth) <= set(idx[b, G].tolist())


# ------------------------------------------------------------------ decode


def _decode_both(svl, orc, wl, cpu, dev, idx, flags=0):
    k = idx.shape[-1]
    lse = torch.empty(wl.B, wl.H, device="cuda")
    out, _ = svl.sparse_decode_attn(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb,
                                    wl.nv, torch.as_tensor(idx).cuda() if k else None,
                                    flags=flags, lse_out=lse)
    torch.cuda.synchronize()
    oo, ol = orc.sparse_decode(cpu["q_dec"], cpu["K"], cpu["V"], cpu["seq_len"], wl.vb, wl.nv,
                               idx if k else np.zeros((wl.B, 1 if flags & 2 else wl.Hkv, 0), np.int32),
                               flags=flags, nthreads=NTH)
    return out.cpu().numpy(), lse.cpu().numpy(), oo, ol


@pytest.mark.parametrize("name", ["toy", "nvila-4k", "long-video", "multi-turn"])
def test_decode_configs(svl, orc, name):
    wl = gen.CONFIGS[name]
    cpu, dev = _gen(wl, seed=11, big=(name != "toy"))
    oi, _, _ = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, wl.k, nthreads=NTH)
    out, lse, oo, ol = _decode_both(svl, orc, wl, cpu, dev, oi)
    mx, rel = parity.check_attention(out, lse, oo, ol)
    print(f"{name}: max-abs {mx:.2e} rel {rel:.2e}")


@pytest.mark.parametrize("B,H,Hkv,d,nv,k,vb,ta", [
    (2, 4, 2, 64, 300, 37, 5, 11), (3, 28, 4, 128, 999, 999, 32, 50), (1, 16, 1, 128, 500, 0, 7, 3),
    (2, 8, 8, 128, 2000, 129, 0, 1), (1, 32, 2, 64, 4096, 700, 64, 300)])
def test_decode_shapes(svl, orc, B, H, Hkv, d, nv, k, vb, ta):
    wl = gen.DecodeWorkload("ds", B, H, Hkv, d, vb, nv, ta, k, 1, 128)
    if B > 1:
        wl.seq_lens = [wl.seq_len - (b * 3) % max(ta, 1) for b in range(B)]
    cpu, dev = _gen(wl, seed=B + k)
    rng = np.random.default_rng(k)
    idx = np.stack([np.stack([np.sort(rng.choice(nv, k, replace=False)) for _ in range(Hkv)])
                    for _ in range(B)]).astype(np.int32)
    out, lse, oo, ol = _decode_both(svl, orc, wl, cpu, dev, idx)
    parity.check_attention(out, lse, oo, ol)


def test_decode_full_selection_equals_dense(svl, orc):
    wl = gen.DecodeWorkload("kd", 2, 28, 4, 128, 32, 3000, 200, 3000, 1, 256)
    cpu, dev = _gen(wl, seed=12)
    idx = np.tile(np.arange(wl.nv, dtype=np.int32), (2, 4, 1))
    out, lse, _, _ = _decode_both(svl, orc, wl, cpu, dev, idx)
    ref, rlse = orc.dense_attn(cpu["q_dec"], cpu["K"], cpu["V"], cpu["seq_len"], nthreads=NTH)
    parity.check_attention(out, lse, ref, rlse)


def test_decode_shared_selection(svl, orc):
    wl = gen.DecodeWorkload("sh", 2, 28, 4, 128, 32, 2048, 64, 200, 1, 256)
    cpu, dev = _gen(wl, seed=13)
    oi, _, _ = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, wl.k, flags=2)
    gi = svl.retrieve(dev["q"], dev["K"], dev["seq_len"], wl.vb, wl.nv, wl.k, flags=2)
    assert gi.shape == (2, 1, 200)
    out, lse, oo, ol = _decode_both(svl, orc, wl, cpu, dev, oi, flags=2)
    parity.check_attention(out, lse, oo, ol)


@pytest.mark.parametrize("early", [0, 1])
def test_decode_bad_indices_flagged(svl, early):
    wl = gen.DecodeWorkload("bad", 1, 8, 2, 64, 4, 300, 10, 20, 1, 64)
    x = gen.make_decode_inputs(wl, seed=14, device="cuda")
    idx = torch.arange(20, dtype=torch.int32, device="cuda").flip(0).expand(1, 2, 20).contiguous()
    ws = svl.Workspace()
    ws.get(1 << 20)
    ws.reset_flags()
    fl = svl.SVL_DECODE_STATIC_PREFIX if early else 0  # (the early gathers resolve the same rows)
    out, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx, flags=fl, ws=ws)
    assert ws.flags() & svl.SVL_DEVFLAG_INDEX
    assert torch.isfinite(out).all()


def test_decode_deterministic_bitwise(svl):
    wl = gen.CONFIGS["long-video"]
    x = gen.make_decode_inputs(wl, seed=15, device="cuda")
    idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k)
    a, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx)
    a = a.clone()
    b, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx)
    assert torch.equal(a, b)


def test_sweep_sampled_rows(svl, orc):
    """Sweep config at full size (B=16, 64k visual): GPU on the whole batch,
    oracle on sampled batch rows."""
    wl = gen.CONFIGS["sweep"]
    x = gen.make_decode_inputs(wl, seed=16, device="cuda")
    sc = torch.empty(wl.B, wl.Hkv, wl.nv, device="cuda")
    idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, scores_out=sc)
    out, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx)
    torch.cuda.synchronize()
    for b in (0, 15):
        q = x["q"][b:b + 1].cpu()
        K = x["K"][b:b + 1].cpu()
        V = x["V"][b:b + 1].cpu()
        sl = x["seq_len"][b:b + 1].cpu()
        oi, osc, gap = orc.retrieve(q, K, sl, wl.vb, wl.nv, wl.k, nthreads=NTH)
        _check_scores(sc[b:b + 1].cpu().numpy(), osc)
        parity.check_indices(idx[b:b + 1].cpu().numpy(), osc, gap, wl.k)
        oo, ol = orc.sparse_decode(x["q_dec"][b:b + 1].cpu(), K, V, sl, wl.vb, wl.nv,
                                   idx[b:b + 1].cpu().numpy(), nthreads=NTH)
        parity.check_attention(out[b:b + 1].cpu().numpy(), None, oo, ol)


# ------------------------------------------------------------------ prune


@pytest.mark.parametrize("ties", [False, True])
def test_prune_per_frame_bitexact(svl, orc, ties):
    B, F, Nf = 2, 256, 512
    sal = gen.make_saliency(B, F * Nf, seed=17, ties=ties)
    offs = list(range(0, F * Nf + 1, Nf))
    gk, gt = svl.prefill_prune(sal.cuda(), 0.75, offs)
    ok, ot = orc.prune(sal.numpy(), 0.75, offs)
    assert gt == ot == 256 * 128
    parity.check_prune(gk.cpu().numpy(), ok)


def test_prune_ragged_and_global(svl, orc):
    sal = gen.make_saliency(3, 131072, seed=18, ties=True)
    sal[1, 5] = -0.0
    sal[1, 6] = 0.0
    gk, gt = svl.prefill_prune(sal.cuda(), 0.9)
    ok, ot = orc.prune(sal.numpy(), 0.9)
    assert gt == ot
    parity.check_prune(gk.cpu().numpy(), ok)
    offs = [0, 1, 1, 700, 5000, 5001, 131072]
    gk, gt = svl.prefill_prune(sal.cuda(), 0.3, offs)
    ok, ot = orc.prune(sal.numpy(), 0.3, offs)
    assert gt == ot
    parity.check_prune(gk.cpu().numpy(), ok)


def test_prune_nan_flagged_and_ranked_lowest(svl):
    sal = torch.rand(1, 1000)
    sal[0, 3] = float("nan")
    ws = svl.Workspace()
    ws.get(4096)
    ws.reset_flags()
    gk, gt = svl.prefill_prune(sal.cuda(), 0.001, ws=ws)   # keep 999 of 1000
    assert ws.flags() & svl.SVL_DEVFLAG_NONFINITE
    assert 3 not in gk.cpu().numpy()[0].tolist()


# ------------------------------------------------------------------ salience


@pytest.mark.parametrize("S,mode,Nf,He,de", [(0, 2, 196, 4, 72), (1, 0, 300, 3, 64),
                                             (4, 1, 129, 2, 128), (0, 2, 512, 16, 72)])
def test_salience_modes(svl, orc, S, mode, Nf, He, de):
    wl = gen.PrefillWorkload("sal", 2, S, Nf, He, de)
    x = gen.make_prefill_inputs(wl, seed=19)
    sal = svl.salience(x["Qe"].cuda(), x["Ke"].cuda(), S, mode)
    ref = orc.salience(x["Qe"], x["Ke"], S, mode, nthreads=NTH)
    parity.check_salience(sal.cpu().numpy(), ref)


def test_salience_then_prune_chain(svl, orc):
    wl = gen.PrefillWorkload("chain", 4, 0, 512, 4, 72)
    x = gen.make_prefill_inputs(wl, seed=20)
    sal = svl.salience(x["Qe"].cuda(), x["Ke"].cuda(), 0, 2)
    ref = orc.salience(x["Qe"], x["Ke"], 0, 2, nthreads=NTH)
    offs = list(range(0, 4 * 512 + 1, 512))
    gk, gt = svl.prefill_prune(sal.reshape(1, -1), 0.75, offs)
    # gap rule on GPU-computed salience (c6): compare against oracle salience per frame
    ok, ot = orc.prune(ref.reshape(1, -1).astype(np.float32), 0.75, offs)
    gk = gk.cpu().numpy()[0]
    for f in range(4):
        s = ref[f]
        sel = gk[(gk >= f * 512) & (gk < (f + 1) * 512)] - f * 512
        order = np.lexsort((np.arange(512), -s))
        gap = (s[order[127]] - s[order[128]]) / s[order[127]]
        parity.check_indices(sel[None, None], s[None, None], np.array([[gap]]), 128)


def test_topk_fallback_massive_ties(svl, orc):
    """Thousands of exact ties in the threshold bin force the cluster radix
    fallback of cluster_topk; ties must still go to the lowest indices."""
    sal = torch.ones(2, 10000)
    sal[1, ::7] = 2.0
    gk, gt = svl.prefill_prune(sal.cuda(), 0.5)
    ok, ot = orc.prune(sal.numpy(), 0.5)
    parity.check_prune(gk.cpu().numpy(), ok)
    assert gk[0].cpu().tolist() == list(range(5000))
    wl = gen.DecodeWorkload("tie", 1, 8, 2, 64, 4, 9000, 6, 3000, 1, 256, sinks=0, needles=0)
    cpu, dev = _gen(wl, seed=21)
    cpu["K"][:, :, 4:9004] = cpu["K"][:, :, 4:5]          # every visual key identical
    dev["K"] = cpu["K"].cuda()
    idx, sc, oi, osc, gap = _retrieve_both(svl, orc, wl, cpu, dev)
    assert np.array_equal(idx, oi)
    assert idx[0, 0].tolist() == list(range(3000))


# ------------------------------------------- many units: relevance pass + refined select
# B * Hkv * CS > 2 CTAs per SM: svl_retrieve runs the relevance pass and the 8192-row-slice
# select (mode 3), whose threshold bin overflows 64 candidates per CTA on these smooth score
# distributions and is narrowed by the refinement round (tools/exp/sanitize_new.py checks the
# path with the A/B flag build).
MANY = gen.DecodeWorkload("many", 10, 28, 4, 128, 32, 16384, 300, 1638, 1, 256)


def test_retrieve_many_units_refined(svl, orc):
    cpu, dev = _gen(MANY, seed=31, big=True)
    idx, sc, oi, osc, gap = _retrieve_both(svl, orc, MANY, cpu, dev)
    _check_scores(sc, osc)
    parity.check_indices(idx, osc, gap, MANY.k)


def test_retrieve_many_units_gapped_exact(svl, orc):
    for gamma in (4.0, 8.0, 16.0):
        wl = gen.DecodeWorkload(**{**MANY.__dict__, "gap_gamma": gamma, "sinks": 0, "needles": 0})
        cpu, dev = _gen(wl, seed=32, big=True)
        idx, sc, oi, osc, gap = _retrieve_both(svl, orc, wl, cpu, dev)
        if gap.min() > 1e-3:
            break
    assert gap.min() > 1e-3, gap.min()
    assert np.array_equal(idx, oi)


def test_retrieve_many_units_duplicates_and_ties(svl, orc):
    cpu, dev = _gen(MANY, seed=33, big=True)
    _, _, oi, osc, _ = _retrieve_both(svl, orc, MANY, cpu, dev)
    for b in (0, 7):
        for G in (0, 3):
            order = np.lexsort((np.arange(MANY.nv), -osc[b, G]))
            kth = int(order[MANY.k - 1])
            for dup in order[MANY.k:MANY.k + 40].tolist()[:6]:  # copies of the k-th key past the cut
                cpu["K"][b, G, MANY.vb + dup] = cpu["K"][b, G, MANY.vb + kth]
    cpu["K"][9, 2, MANY.vb:MANY.vb + MANY.nv] = cpu["K"][9, 2, MANY.vb]  # a unit of identical keys
    dev["K"] = cpu["K"].cuda()
    idx, sc, oi, osc, gap = _retrieve_both(svl, orc, MANY, cpu, dev)
    assert np.array_equal(idx, oi)                      # exact at gap 0: ties to the lower index
    assert idx[9, 2].tolist() == list(range(MANY.k))
