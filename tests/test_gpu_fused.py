"""GPU parity of svl_fresh_decode_step (fused retrieve + sparse decode) vs the
fp64 oracle: indices by the gap rule, attention output within tolerance
(SURVEY.md 8(c) c6), at toy size and the BASELINE configs at full size."""
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


def _run(svl, orc, wl, seed, flags=0, k=None, big=True, xflags=0):
    """fresh step vs the oracle; xflags = library-only flags (SVL_PIN_SPLITS, SVL_FRESH_UNFUSED)"""
    k = wl.k if k is None else k
    x = gen.make_decode_inputs(wl, seed=seed, device="cuda" if big else "cpu")
    cpu = {kk: v.cpu() for kk, v in x.items()}
    dev = {kk: v.cuda() for kk, v in x.items()}
    lse = torch.empty(wl.B, wl.H, device="cuda")
    out, idx = svl.fresh_decode_step(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb,
                                     wl.nv, k, flags=flags | xflags, lse_out=lse)
    torch.cuda.synchronize()
    idx = idx.cpu().numpy()
    oi, osc, gap = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, k, flags=flags,
                                nthreads=NTH)
    frac = parity.check_indices(idx, osc, gap, k)
    # decode parity on the GPU's own (validated) selection
    oo, ol = orc.sparse_decode(cpu["q_dec"], cpu["K"], cpu["V"], cpu["seq_len"], wl.vb, wl.nv,
                               idx if k else np.zeros((wl.B, wl.Hkv, 0), np.int32), nthreads=NTH)
    mx, rel = parity.check_attention(out.cpu().numpy(), lse.cpu().numpy(), oo, ol)
    return frac, mx, rel, idx, oi


@pytest.mark.parametrize("name", ["toy", "nvila-4k", "long-video", "multi-turn"])
@pytest.mark.parametrize("flags", [0, 1])
def test_fresh_step_configs(svl, orc, name, flags):
    wl = gen.CONFIGS[name]
    frac, mx, rel, _, _ = _run(svl, orc, wl, seed=31, flags=flags, big=(name != "toy"))
    print(f"{name} flags={flags}: strict {frac:.2f} max-abs {mx:.2e} rel {rel:.2e}")


def test_fresh_step_gapped_bitexact(svl, orc):
    base = gen.CONFIGS["long-video"]
    for gamma in (4.0, 8.0, 16.0):
        wl = gen.DecodeWorkload(**{**base.__dict__, "gap_gamma": gamma, "sinks": 0, "needles": 0})
        x = gen.make_decode_inputs(wl, seed=32, device="cuda")
        oi, osc, gap = orc.retrieve(x["q"].cpu(), x["K"].cpu(), x["seq_len"].cpu(), wl.vb, wl.nv,
                                    wl.k, nthreads=NTH)
        if gap.min() > 1e-3:
            break
    out, idx = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
    assert np.array_equal(idx.cpu().numpy(), oi)


@pytest.mark.parametrize("k", [12288, 20000])
def test_fresh_step_overflow_batches(svl, orc, k):
    """Stage-1 split pipeline with more kept rows per CTA than its V staging holds (3/8 and
    ~5/8 of 32k visual rows kept, gapped so the threshold bin stays small): the decode warps
    run overflow batches (P rows re-read from TMEM) before the candidates; indices exact,
    attention within tolerance."""
    base = gen.CONFIGS["long-video"]
    for gamma in (6.0, 10.0, 16.0):
        wl = gen.DecodeWorkload(**{**base.__dict__, "name": "ovf", "k": k, "gap_gamma": gamma, "sinks": 0,
                                   "needles": 0})
        x = gen.make_decode_inputs(wl, seed=71, device="cpu")
        oi, osc, gap = orc.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, k, nthreads=NTH)
        if gap.min() > 1e-3:
            break
    frac, mx, rel, idx, oi2 = _run(svl, orc, wl, seed=71)
    assert np.array_equal(idx, oi)


@pytest.mark.parametrize("kfrac", [0.5, 0.97, "nv-1"])
def test_fresh_step_large_k(svl, orc, kfrac):
    """Most of the visual rows kept (the threshold bin near the bottom of the value range;
    above-b* rows overflow the staging): indices by the gap rule, attention within tolerance."""
    base = gen.CONFIGS["nvila-4k"]
    k = base.nv - 1 if kfrac == "nv-1" else int(base.nv * kfrac)
    wl = gen.DecodeWorkload(**{**base.__dict__, "name": "lk", "k": k})
    _run(svl, orc, wl, seed=81, k=k)


@pytest.mark.parametrize("k", [0, 1, 2000])
def test_fresh_step_k_edges_ragged(svl, orc, k):
    wl = gen.DecodeWorkload("fe", 3, 28, 4, 128, 19, 2000, 77, k, 1, 256)
    wl.seq_lens = [wl.seq_len, wl.seq_len - 30, wl.seq_len - 70]
    _run(svl, orc, wl, seed=33 + k, k=k, big=False)


@pytest.mark.parametrize("H,Hkv,d", [(16, 1, 128), (8, 2, 64), (4, 4, 64), (32, 2, 128)])
def test_fresh_step_shapes(svl, orc, H, Hkv, d):
    wl = gen.DecodeWorkload("fs", 2, H, Hkv, d, 8, 5000, 40, 500, 1, 256)
    _run(svl, orc, wl, seed=34, big=False)


def test_fresh_step_matches_unfused(svl):
    """Fused == retrieve + sparse decode (the two-call path) within tolerance,
    identical kept sets where the selection is not a near-tie."""
    wl = gen.CONFIGS["long-video"]
    x = gen.make_decode_inputs(wl, seed=35, device="cuda")
    out_f, idx_f = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
    idx_u = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k)
    out_u, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx_u)
    torch.cuda.synchronize()
    same = (idx_f == idx_u).all(dim=-1).float().mean().item()
    assert same >= 0.5
    if same == 1.0:
        assert (out_f - out_u).abs().max().item() < 1e-5


def test_fresh_step_sweep_fallback_sampled(svl, orc):
    """64k visual tokens exceed the fused on-chip budget -> the two-call path."""
    wl = gen.CONFIGS["sweep"]
    x = gen.make_decode_inputs(wl, seed=36, device="cuda")
    out, idx = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
    torch.cuda.synchronize()
    for b in (3,):
        sl = slice(b, b + 1)
        cpu = {kk: v[sl].cpu() for kk, v in x.items()}
        oi, osc, gap = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, wl.k, nthreads=NTH)
        parity.check_indices(idx[sl].cpu().numpy(), osc, gap, wl.k)
        oo, ol = orc.sparse_decode(cpu["q_dec"], cpu["K"], cpu["V"], cpu["seq_len"], wl.vb, wl.nv,
                                   idx[sl].cpu().numpy(), nthreads=NTH)
        parity.check_attention(out[sl].cpu().numpy(), None, oo, ol)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_fresh_step_simulated_shards_bitwise(svl, P):
    """SURVEY.md 4 'simulated-shard test': each rank's (batch x KV-head) slice
    run separately on one GPU and assembled == the unsharded run, bitwise, with
    the per-unit split count pinned -- the planner may pick
    a different cluster size for a different number of units."""
    from paper_2510_17777_b200 import sharding
    pin = svl.SVL_PIN_SPLITS(8)
    wl = gen.DecodeWorkload("shd", 4, 28, 4, 128, 32, 8192, 300, 819, 1, 256)
    x = gen.make_decode_inputs(wl, seed=38, device="cuda")
    ref, _ = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, flags=pin)
    ref = ref.clone()
    parts, plans = [], []
    for r in range(P):
        sp = sharding.plan(wl.B, wl.H, wl.Hkv, P, r)
        ql, Kl, Vl, sl = sharding.local_inputs(sp, x["q_dec"], x["K"], x["V"], x["seq_len"])
        o, _ = svl.fresh_decode_step(ql, Kl, Vl, sl, wl.vb, wl.nv, wl.k, flags=pin)
        parts.append(o.clone())
        plans.append(sp)
    full = sharding.assemble(parts, plans, wl.B, wl.H)
    assert torch.equal(full, ref)


def test_fresh_step_deterministic(svl):
    wl = gen.CONFIGS["long-video"]
    x = gen.make_decode_inputs(wl, seed=37, device="cuda")
    a, ia = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
    a, ia = a.clone(), ia.clone()
    b, ib = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
    assert torch.equal(a, b) and torch.equal(ia, ib)


@pytest.mark.parametrize("pin", [None, "16"])
@pytest.mark.parametrize("B,nv", [(2, 32768), (3, 32768), (5, 24576), (8, 32768), (8, 24576)])
def test_fresh_step_many_units(svl, orc, B, nv, pin):
    """More clusters than fit at once (later clusters start on SMs vacated by earlier
    ones): this exposed the text-row / ring-slot parity race fixed in fused.cu (the
    text rows now have their own buffer and barrier); run twice back to back.  B = 3 at 32k
    and B = 5 at 24k take the fused kernel unpinned (the planner's up-to-three-wave rule)."""
    # pin: force the fused kernel into a multi-wave launch (the planner would take two calls)
    xf = svl.SVL_PIN_SPLITS(int(pin)) if pin else 0
    base = gen.CONFIGS["long-video"]
    wl = gen.DecodeWorkload(**{**base.__dict__, "name": f"mu{B}", "B": B, "nv": nv, "k": nv // 10,
                               "seq_lens": None})
    _run(svl, orc, wl, seed=40 + B, xflags=xf)
    _run(svl, orc, wl, seed=41 + B, xflags=xf)


def test_multi_turn_eviction_is_a_seq_len_rollback(svl):
    """SURVEY.md 8(f) f4(ii) / SPEC.md:306-314 evict_round: evicting a round's question and
    answer rows (multi-turn) is a seq_len rollback of the after-visual text.
    Append a round (new K/V rows past seq_len), decode, roll seq_len back: the fresh step is
    bitwise the pre-round one (the visual cache and everything below seq_len untouched)."""
    wl = gen.CONFIGS["multi-turn"]
    x = gen.make_decode_inputs(wl, seed=61, device="cuda")
    a, ia = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
    a, ia = a.clone(), ia.clone()
    room = wl.capacity - int(x["seq_len"].max())
    n_round = min(12, room)
    assert n_round > 0
    g = torch.Generator(device="cuda").manual_seed(62)
    for b in range(wl.B):  # the round's rows: written past each batch row's seq_len
        L = int(x["seq_len"][b])
        x["K"][b, :, L:L + n_round] = torch.randn(wl.Hkv, n_round, wl.d, generator=g, device="cuda").to(torch.bfloat16)
        x["V"][b, :, L:L + n_round] = torch.randn(wl.Hkv, n_round, wl.d, generator=g, device="cuda").to(torch.bfloat16)
    longer = (x["seq_len"] + n_round).to(torch.int32)
    c, ic = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], longer, wl.vb, wl.nv, wl.k)
    assert not torch.equal(c, a)  # the round's rows are attended
    b_, ib = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
    assert torch.equal(b_, a) and torch.equal(ib, ia)
