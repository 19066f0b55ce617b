"""Sequence-split fresh step simulated on one GPU:
P_s shard views, the three exchanges as stacks, every step in the library's
kernels.  Kept sets vs the fp64 oracle by the gap rule (reading c6), output and
LSE within the attention tolerance, and the unsharded fused step agrees."""
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


@pytest.mark.parametrize("name,P_s", [("long-video", 2), ("long-video", 4), ("nvila-4k", 2), ("toy", 2)])
def test_seq_split_vs_oracle(svl, orc, name, P_s):
    from paper_2510_17777_b200 import seqpar
    wl = gen.CONFIGS[name]
    x = gen.make_decode_inputs(wl, seed=61 + P_s)
    dev = {kk: v.cuda() for kk, v in x.items()}
    out, lse, idx = seqpar.simulated_step(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, wl.k, P_s)
    torch.cuda.synchronize()
    oi, osc, gap = orc.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, nthreads=NTH)
    frac = parity.check_indices(idx.cpu().numpy(), osc, gap, wl.k)
    oo, ol = orc.sparse_decode(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx.cpu().numpy(),
                               nthreads=NTH)
    parity.check_attention(out.cpu().numpy(), lse.cpu().numpy(), oo, ol)
    f_out, f_idx = svl.fresh_decode_step(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, wl.k)
    torch.cuda.synchronize()
    if torch.equal(f_idx, idx):
        assert (f_out - out).abs().max().item() < 1e-4
    print(f"{name} P_s={P_s}: strict {frac:.2f}")


def test_seq_split_ragged_batch(svl, orc):
    from paper_2510_17777_b200 import seqpar
    wl = gen.DecodeWorkload("sp-rag", 2, 28, 4, 128, 32, 8192, 200, 819, 1, 256)
    wl.seq_lens = [wl.seq_len, wl.seq_len - 77]
    x = gen.make_decode_inputs(wl, seed=66)
    dev = {kk: v.cuda() for kk, v in x.items()}
    out, lse, idx = seqpar.simulated_step(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, wl.k, 2)
    torch.cuda.synchronize()
    oi, osc, gap = orc.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, nthreads=NTH)
    parity.check_indices(idx.cpu().numpy(), osc, gap, wl.k)
    oo, ol = orc.sparse_decode(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx.cpu().numpy(),
                               nthreads=NTH)
    parity.check_attention(out.cpu().numpy(), lse.cpu().numpy(), oo, ol)


def test_primitives(svl):
    """svl_lse_combine / svl_merge_partials / svl_shard_indices / svl_topk on small cases
    against their definitions (float64 numpy)."""
    g = torch.Generator(device="cuda").manual_seed(1)
    parts = torch.randn(3, 5, 7, device="cuda", generator=g) * 4
    got = svl.lse_combine(parts)
    ref = torch.logsumexp(parts.double(), dim=0)
    assert (got.double() - ref).abs().max().item() < 1e-5
    outs = torch.randn(3, 5, 7, 16, device="cuda", generator=g)
    o, l = svl.merge_partials(outs, parts)
    w = torch.softmax(parts.double(), dim=0)
    assert (o.double() - (w[..., None] * outs.double()).sum(0)).abs().max().item() < 1e-5
    assert (l.double() - ref).abs().max().item() < 1e-5
    idx = torch.tensor([[1, 5, 9, 12, 20, 31]], dtype=torch.int32, device="cuda")
    assert svl.shard_indices(idx, 8, 16).tolist() == [[1, 4, -1, -1, -1, -1]]
    assert svl.shard_indices(idx, 16, 32).tolist() == [[4, 15, -1, -1, -1, -1]]
    sc = torch.tensor([[0.3, 0.1, 0.3, 0.5, 0.5, 0.0]], device="cuda")
    assert svl.topk(sc, 3).tolist() == [[0, 3, 4]]
