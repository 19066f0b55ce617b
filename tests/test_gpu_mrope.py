"""svl_mrope_remap (multimodal-RoPE remap after pruning, SURVEY.md 8(f) f4(i);
PAPER.md:127; reading A23) vs the fp64 oracle: the plan
(per-dimension ranks, text start) exact, every re-rotated key within one bf16
ulp of the exact value, V rows copied bit-exactly; diagonal coordinates give
the unified remap bitwise; bad coordinates are flagged."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def svl():
    from paper_2510_17777_b200 import build, svl as mod
    build.build()
    mod.lib()
    return mod


def _video_case(B, Hkv, d, vb, T, Hg, Wg, ta, keep, seed):
    """Frames T x grid Hg x Wg of visual tokens with (t, h, w) coordinates, a random kept set."""
    g = torch.Generator().manual_seed(seed)
    nv = T * Hg * Wg
    cap = vb + nv + ta + 5
    K = torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16)
    V = torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16)
    t, h, w = torch.meshgrid(torch.arange(T), torch.arange(Hg), torch.arange(Wg), indexing="ij")
    coords = torch.stack([t.reshape(-1), h.reshape(-1), w.reshape(-1)], -1).to(torch.int32)
    coords = coords.unsqueeze(0).expand(B, nv, 3).contiguous()
    kept = torch.stack([torch.sort(torch.randperm(nv, generator=g)[:keep]).values for _ in range(B)]).to(torch.int32)
    seq = torch.tensor([vb + nv + ta - 2 * b for b in range(B)], dtype=torch.int32)
    return K, V, coords, kept, seq, nv


def _ulp_check(got, exact):
    ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(exact), 2.0 ** -126))) - 7)
    assert (np.abs(got - exact) <= ulp).all(), np.abs(got - exact).max()


@pytest.mark.parametrize("B,Hkv,d,vb,T,Hg,Wg,ta,keep,sec,base", [
    (1, 2, 64, 6, 4, 8, 8, 12, 64, (8, 12, 12), 10000.0),
    (2, 4, 128, 32, 16, 16, 16, 300, 1024, (16, 24, 24), 1000000.0),      # Qwen2-VL sections
    (1, 4, 128, 32, 128, 16, 16, 768, 8192, (16, 24, 24), 1000000.0),     # long video, 25 % kept
])
def test_mrope_remap_parity(svl, orc, B, Hkv, d, vb, T, Hg, Wg, ta, keep, sec, base):
    K, V, coords, kept, seq, nv = _video_case(B, Hkv, d, vb, T, Hg, Wg, ta, keep, seed=T * Hg)
    Ko, Vo, nc, ts = svl.mrope_remap(K.cuda(), V.cuda(), seq.cuda(), vb, nv, coords.cuda(), kept.cuda(), base, sec)
    torch.cuda.synchronize()
    onc, ots = orc.mrope_plan(coords.numpy(), vb, kept.numpy())
    assert np.array_equal(nc.cpu().numpy(), onc) and np.array_equal(ts.cpu().numpy(), ots)
    ref, rows = orc.mrope_remap(K, seq.numpy(), vb, nv, kept.numpy(), onc, ots, sec, base, cap_out=Ko.shape[2])
    Ko, Vo = Ko.cpu(), Vo.cpu()
    for b in range(B):
        n = int(seq[b]) - nv + keep
        _ulp_check(Ko[b, :, :n].double().numpy(), ref[b, :, :n])
        assert torch.equal(Vo[b, :, :n], V[b][:, torch.as_tensor(rows[b][:n]).long()])


def test_mrope_diagonal_equals_unified(svl):
    """(i, i, i) coordinates: the mRoPE remap is the unified remap, bitwise."""
    g = torch.Generator().manual_seed(9)
    B, Hkv, d, vb, nv, ta, k = 1, 2, 128, 16, 600, 40, 150
    cap = vb + nv + ta
    K = torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16).cuda()
    V = torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16).cuda()
    seq = torch.tensor([cap], dtype=torch.int32, device="cuda")
    coords = torch.arange(nv, dtype=torch.int32).view(1, nv, 1).expand(1, nv, 3).contiguous().cuda()
    kept = torch.sort(torch.randperm(nv, generator=g)[:k]).values.to(torch.int32).view(1, k).cuda()
    a, av, _, ts = svl.mrope_remap(K, V, seq, vb, nv, coords, kept, 1000000.0, (16, 24, 24))
    b, bv, seq_new = svl.rope_remap(K, V, seq, vb, nv, kept, 1000000.0)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(av, bv) and int(ts[0]) == vb + k


def test_mrope_bad_coordinate_flagged(svl):
    K, V, coords, kept, seq, nv = _video_case(1, 1, 64, 4, 2, 4, 4, 6, 10, seed=1)
    coords[0, int(kept[0, 3]), 1] = 70000
    ws = svl.Workspace()
    ws.get(svl.lib().svl_mrope_remap_workspace_size(1, 10))
    ws.reset_flags()
    svl.mrope_remap(K.cuda(), None, seq.cuda(), 4, nv, coords.cuda(), kept.cuda(), 10000.0, (8, 12, 12), ws=ws)
    assert ws.flags() & svl.SVL_DEVFLAG_INDEX
