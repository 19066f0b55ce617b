"""Ties on the headline path: svl_fresh_decode_step at long-video size
(B = 1, 32768 visual rows, k = 3277 -- the fused kernel) with exact duplicate
keys across the k-boundary (reading A21; SPEC.md:248,
265), every visual key equal, and quantised keys with thousands of exact ties
per value.  The last two put more than 64 keys of the threshold bin into one
CTA, so the fused kernel's stage-2 generic exact radix (fused.cu, stage == 2:
text V re-gathered after the cluster barrier) decides the set.  Ties go to the
lower index on both sides: wherever the oracle's scores tie exactly, the GPU
set must be exactly the oracle's; elsewhere the gap rule (tests/parity.py)."""
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


def _fresh_vs_oracle(svl, orc, wl, cpu, flags=0):
    dev = {kk: v.cuda() for kk, v in cpu.items()}
    lse = torch.empty(wl.B, wl.H, device="cuda")
    out, idx = svl.fresh_decode_step(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv,
                                     wl.k, flags=flags, lse_out=lse)
    torch.cuda.synchronize()
    idx = idx.cpu().numpy()
    oi, osc, gap = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, wl.k, nthreads=NTH)
    parity.check_indices(idx, osc, gap, wl.k)
    oo, ol = orc.sparse_decode(cpu["q_dec"], cpu["K"], cpu["V"], cpu["seq_len"], wl.vb, wl.nv, idx,
                               nthreads=NTH)
    parity.check_attention(out.cpu().numpy(), lse.cpu().numpy(), oo, ol)
    return idx, oi, osc


def _lv(**kw):
    base = gen.CONFIGS["long-video"]
    return gen.DecodeWorkload(**{**base.__dict__, "name": "lv-ties", **kw})


@pytest.mark.parametrize("flags_name", ["fused", "unfused"])
def test_fresh_duplicates_across_k_boundary(svl, orc, flags_name):
    """The k-th row (oracle order) copied into unselected rows before and after it:
    among identical rows the lower indices win, on the fused and the two-call path.
    Copying rows changes each head's log-sum-exp (FULL_PREFIX), which moves the
    boundary, so the copy is repeated from the new k-th row until the group of
    identical rows straddles the cut (selected and unselected members)."""
    flags = svl.SVL_FRESH_UNFUSED if flags_name == "unfused" else 0
    wl = _lv()
    cpu = gen.make_decode_inputs(wl, seed=71)
    dups = {}
    for it in range(8):
        oi, osc, _ = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, wl.k, nthreads=NTH)
        straddle = 0
        for G in range(wl.Hkv):
            if G in dups:
                kept = np.isin(dups[G], oi[0, G])
                if kept.any() and not kept.all():
                    straddle += 1
                    continue
            order = np.lexsort((np.arange(wl.nv), -osc[0, G]))
            kth = int(order[wl.k - 1])
            first = [int(j) for j in order[wl.k:wl.k + 400] if abs(int(j) - kth) > 64][:8]
            dups[G] = sorted(set(dups.get(G, first)) | {kth})
            for j in dups[G]:
                cpu["K"][0, G, wl.vb + j] = cpu["K"][0, G, wl.vb + kth]
        if straddle == wl.Hkv:
            break
    assert straddle >= wl.Hkv - 1, "the duplicate groups do not straddle the cut"
    idx, oi, osc = _fresh_vs_oracle(svl, orc, wl, cpu, flags)
    for G in range(wl.Hkv):
        members = dups[G]
        rows = cpu["K"][0, G, wl.vb + torch.as_tensor(members)]
        assert bool((rows == rows[:1]).all())  # identical rows
        sel = [j for j in members if j in set(idx[0, G].tolist())]
        # the duplicates tie exactly: whichever count is kept, it is the lowest indices
        assert sel == members[:len(sel)], (G, members, sel)
        assert np.array_equal(np.isin(members, idx[0, G]), np.isin(members, oi[0, G]))


def test_fresh_all_visual_keys_equal(svl, orc):
    """Every visual relevance score identical: the kept set is rows [0, k), and the
    selection goes through the fused kernel's generic-radix fallback (stage 2)."""
    wl = _lv(sinks=0, needles=0)
    cpu = gen.make_decode_inputs(wl, seed=72)
    cpu["K"][:, :, wl.vb:wl.vb + wl.nv] = cpu["K"][:, :, wl.vb:wl.vb + 1]
    idx, oi, _ = _fresh_vs_oracle(svl, orc, wl, cpu)
    for G in range(wl.Hkv):
        assert idx[0, G].tolist() == list(range(wl.k))
    assert np.array_equal(idx, oi)


@pytest.mark.parametrize("levels", [3, 16])
def test_fresh_quantised_massive_ties(svl, orc, levels):
    """Visual keys drawn from `levels` distinct rows: each relevance value is shared by
    ~32768 / levels rows, the threshold bin holds thousands of exact ties (stage 2),
    and the set must be exactly the oracle's (ties to the lower index)."""
    wl = _lv(sinks=0, needles=0)
    cpu = gen.make_decode_inputs(wl, seed=73 + levels)
    rng = np.random.default_rng(levels)
    pick = torch.from_numpy(rng.integers(0, levels, size=wl.nv))
    for G in range(wl.Hkv):
        protos = cpu["K"][0, G, wl.vb:wl.vb + levels].clone()
        cpu["K"][0, G, wl.vb:wl.vb + wl.nv] = protos[pick]
    idx, oi, osc = _fresh_vs_oracle(svl, orc, wl, cpu)
    assert np.array_equal(idx, oi)


def test_fresh_ties_repeatable_and_flag_clean(svl):
    """The stage-2 path twice back to back: bitwise identical, no device flag raised."""
    wl = _lv(sinks=0, needles=0)
    x = gen.make_decode_inputs(wl, seed=74, device="cuda")
    x["K"][:, :, wl.vb:wl.vb + wl.nv] = x["K"][:, :, wl.vb:wl.vb + 1]
    ws = svl.Workspace()
    a, ia = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
    a, ia = a.clone(), ia.clone()
    b, ib = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
    assert torch.equal(a, b) and torch.equal(ia, ib)
    assert ws.flags() == 0
