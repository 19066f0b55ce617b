"""Pack-once (svl_pack_kv): the packed cache holds
exactly the attended rows in order, and decode over it is bitwise the decode over
the original cache with the gathered selection (same rows, same order, same splits)."""
import numpy as np
import pytest
import torch

from paper_2510_17777_b200 import inputs as gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def svl():
    from paper_2510_17777_b200 import build, svl as mod
    build.build()
    mod.lib()
    return mod


@pytest.mark.parametrize("name", ["toy", "nvila-4k", "long-video", "multi-turn"])
def test_pack_rows_and_decode_bitwise(svl, name):
    wl = gen.CONFIGS[name]
    x = gen.make_decode_inputs(wl, seed=51, device="cuda")
    idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k)
    Kp, Vp, slp = svl.pack_kv(x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx)
    torch.cuda.synchronize()
    # rows: the attended rows of the original cache, in order (torch indexing reference)
    for b in range(wl.B):
        L = int(x["seq_len"][b])
        for G in range(wl.Hkv):
            rows = torch.cat([torch.arange(wl.vb, device="cuda"), wl.vb + idx[b, G].long(),
                              torch.arange(wl.vb + wl.nv, L, device="cuda")])
            n = rows.numel()
            assert torch.equal(Kp[b, G, :n], x["K"][b, G, rows])
            assert torch.equal(Vp[b, G, :n], x["V"][b, G, rows])
    # decode over the packed cache == decode over the original with the selection
    ident = torch.arange(wl.k, dtype=torch.int32, device="cuda").expand(wl.B, wl.Hkv, wl.k).contiguous()
    o1, l1 = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx,
                                    lse_out=torch.empty(wl.B, wl.H, device="cuda"))
    o2, l2 = svl.sparse_decode_attn(x["q_dec"], Kp, Vp, slp, wl.vb, wl.k, ident,
                                    lse_out=torch.empty(wl.B, wl.H, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


def test_pack_bad_indices_flagged(svl):
    wl = gen.CONFIGS["toy"]
    x = gen.make_decode_inputs(wl, seed=52, device="cuda")
    idx = torch.arange(wl.k, dtype=torch.int32, device="cuda").expand(wl.B, wl.Hkv, wl.k).contiguous().clone()
    idx[0, 0, 3] = idx[0, 0, 2]  # not strictly ascending
    ws = svl.Workspace()
    ws.get(1024)
    ws.reset_flags()
    svl.pack_kv(x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx, ws=ws)
    assert ws.flags() & svl.SVL_DEVFLAG_INDEX
