"""Parity of the tensor-core retrieve path (svl_retrieve with n_q * g > 32,
SURVEY.md 8(f) f1: question-chunk retrieval) against the fp64
oracle: scores within the retrieve tolerance, indices by the gap rule
(SURVEY.md 8(c) c6), on FULL_PREFIX / VISUAL_ONLY / SHARED / lse_in, d = 64 and
128, ragged seq_len and visual spans that are not multiples of the tiles."""
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


def _run(svl, orc, wl, seed, flags=0, lse=None):
    x = gen.make_decode_inputs(wl, seed=seed, device="cpu")
    cpu = {k: v.cpu() for k, v in x.items()}
    dev = {k: v.cuda() for k, v in x.items()}
    U = 1 if flags & svl.SVL_SELECT_SHARED else wl.Hkv
    sc = torch.empty(wl.B, U, wl.nv, dtype=torch.float32, device="cuda")
    lse_dev = None if lse is None else torch.as_tensor(lse, dtype=torch.float32).cuda()
    idx = svl.retrieve(dev["q"], dev["K"], dev["seq_len"], wl.vb, wl.nv, wl.k, flags=flags,
                       lse_in=lse_dev, scores_out=sc)
    torch.cuda.synchronize()
    oi, osc, gap = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, wl.k, flags=flags,
                                lse_in=lse, nthreads=NTH)
    sc = sc.cpu().numpy()
    err = np.abs(sc - osc) / np.maximum(np.abs(osc), 1e-30)
    big = osc > osc.max() * 1e-6
    assert err[big].max() < 2e-5, err[big].max()
    parity.check_indices(idx.cpu().numpy(), osc, gap, wl.k)
    return cpu, idx, sc


@pytest.mark.parametrize("B,H,Hkv,d,vb,nv,ta,k,n_q", [
    (1, 28, 4, 128, 32, 4096, 300, 1024, 32),   # NVILA-shaped, 224 query rows (one padded block)
    (2, 28, 4, 128, 32, 3000, 300, 300, 64),    # 448 rows: 4 query blocks, 2 N-stages; ragged N_v
    (1, 16, 2, 64, 8, 2000, 200, 200, 8),       # d = 64, 64 rows
    (1, 4, 1, 128, 16, 1500, 600, 150, 130),    # g = 4, 520 rows: 3 N-stages, 5 query blocks
])
@pytest.mark.parametrize("flags", [0, 1])
def test_retrieve_tc_shapes(svl, orc, B, H, Hkv, d, vb, nv, ta, k, n_q, flags):
    wl = gen.DecodeWorkload("tc", B, H, Hkv, d, vb, nv, ta, k, n_q, 256)
    _run(svl, orc, wl, seed=11 + n_q, flags=flags)


def test_retrieve_tc_ragged_seq_len(svl, orc):
    wl = gen.DecodeWorkload("tcr", 3, 28, 4, 128, 32, 2500, 400, 250, 40, 256)
    wl.seq_lens = [wl.seq_len, wl.seq_len - 150, wl.seq_len - 400 + 40]
    _run(svl, orc, wl, seed=3)


def test_retrieve_tc_shared(svl, orc):
    wl = gen.DecodeWorkload("tcs", 2, 28, 4, 128, 32, 2048, 200, 256, 16, 256)
    _run(svl, orc, wl, seed=4, flags=svl.SVL_SELECT_SHARED)


def test_retrieve_tc_lse_in(svl, orc):
    wl = gen.DecodeWorkload("tcl", 1, 28, 4, 128, 32, 2000, 100, 200, 12, 256)
    x = gen.make_decode_inputs(wl, seed=5, device="cpu")
    q, K = x["q"].double(), x["K"].double()
    L = wl.seq_len
    lse = torch.zeros(1, wl.n_q, 28, dtype=torch.float64)
    for r in range(wl.n_q):   # full-prefix LSE from torch float64 (independent of the oracle)
        s = torch.einsum("hjc,hc->hj", K[0].repeat_interleave(7, 0)[:, :L - wl.n_q + r + 1], q[0, r]) / math.sqrt(128)
        lse[0, r] = torch.logsumexp(s, 1)
    _run(svl, orc, wl, seed=5, lse=lse.numpy())


def test_retrieve_tc_gapped_strict(svl, orc):
    """Gapped input (every unit's k/(k+1) gap >= 1e-3): indices must equal the oracle's."""
    wl = gen.DecodeWorkload("tcg", 1, 28, 4, 128, 32, 4096, 200, 512, 32, 256, gap_gamma=4.0)
    cpu, idx, _ = _run(svl, orc, wl, seed=6)
    oi, _, gap = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, wl.k, nthreads=NTH)
    if (gap > 1e-4).all():
        assert np.array_equal(idx.cpu().numpy(), oi)


def test_retrieve_tc_deterministic(svl):
    wl = gen.DecodeWorkload("tcd", 1, 28, 4, 128, 32, 4096, 300, 1024, 32, 256)
    x = gen.make_decode_inputs(wl, seed=8, device="cuda")
    outs = []
    for _ in range(2):
        sc = torch.empty(1, 4, wl.nv, dtype=torch.float32, device="cuda")
        idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, scores_out=sc)
        outs.append((idx.clone(), sc.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_retrieve_tc_four_wave_row_lse_branch(svl, orc):
    """n_q = 512 question rows (3584 per KV group, 28 query blocks): the row-LSE pass takes
    the planner's 4-wave branch (units x query blocks x 2 >= SMs) that the bench's n_q = 512
    run uses (retrieve_tc.cu plan_retrieve_tc); FULL_PREFIX, scores and indices vs the oracle."""
    wl = gen.DecodeWorkload("tc4w", 1, 28, 4, 128, 32, 4096, 600, 1024, 512, 256)
    _run(svl, orc, wl, seed=77)
