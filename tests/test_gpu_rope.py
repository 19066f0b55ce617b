"""svl_rope_remap (unified RoPE remap after pruning)
vs the fp64 oracle: every rotated key within one bf16 ulp of the exact value, V rows
copied bit-exactly, rows past the compacted length untouched; bad kept indices flagged."""
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


def _case(B, Hkv, d, vb, nv, ta, k, seed):
    g = torch.Generator().manual_seed(seed)
    cap = vb + nv + ta + 7
    K = torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16)
    V = torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16)
    kept = torch.stack([torch.sort(torch.randperm(nv, generator=g)[:k]).values for _ in range(B)]).to(torch.int32)
    seq = torch.tensor([vb + nv + ta - 3 * b for b in range(B)], dtype=torch.int32)
    return K, V, kept, seq


@pytest.mark.parametrize("B,Hkv,d,vb,nv,ta,k,base", [
    (1, 2, 64, 8, 512, 24, 128, 10000.0),          # toy-sized
    (2, 4, 128, 32, 4096, 300, 1024, 1000000.0),   # NVILA-shaped, Qwen2 base
    (1, 4, 128, 32, 131072, 768, 32768, 1000000.0),  # the prune bench: 131072 -> 32768 kept
])
def test_rope_remap_parity(svl, orc, B, Hkv, d, vb, nv, ta, k, base):
    K, V, kept, seq = _case(B, Hkv, d, vb, nv, ta, k, seed=nv)
    Ko, Vo, seq_new = svl.rope_remap(K.cuda(), V.cuda(), seq.cuda(), vb, nv, kept.cuda(), base)
    torch.cuda.synchronize()
    ref, rows = orc.rope_remap(K, seq.numpy(), vb, nv, kept.numpy(), base, cap_out=Ko.shape[2])
    Ko, Vo = Ko.cpu(), Vo.cpu()
    for b in range(B):
        n = int(seq_new[b])
        assert n == int(seq[b]) - nv + k and (rows[b][:n] >= 0).all() and (rows[b][n:] == -1).all()
        got = Ko[b, :, :n].double().numpy()
        exact = ref[b, :, :n]
        # one bf16 ulp of the exact value (2^(floor(log2|x|) - 7)), tiny values: 2^-133
        ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(exact), 2.0 ** -126))) - 7)
        assert (np.abs(got - exact) <= ulp).all(), np.abs(got - exact).max()
        assert torch.equal(Vo[b, :, :n], V[b][:, torch.as_tensor(rows[b][:n]).long()])
        assert (Ko[b, :, n:] == 0).all() and (Vo[b, :, n:] == 0).all()


def test_rope_remap_bad_kept_flagged(svl):
    K, V, kept, seq = _case(1, 1, 64, 4, 64, 8, 16, seed=3)
    kept[0, 5] = kept[0, 4]
    ws = svl.Workspace()
    ws.get(1024)
    ws.reset_flags()
    svl.rope_remap(K.cuda(), None, seq.cuda(), 4, 64, kept.cuda(), 10000.0, ws=ws)
    assert ws.flags() & svl.SVL_DEVFLAG_INDEX
