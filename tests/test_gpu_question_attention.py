"""Parity of svl_question_attention (the question chunk's
attention output on the tensor cores) against the fp64 oracle.

Bound (reading A24): P is rounded to bf16 before the P.V product, so
|out - ref| <= 2^-9 * sum_j P_j |V_j| per element, plus the fp32 logits and
accumulation; the test allows 2^-8 * absmass + 1e-5.  LSE within 2e-4 (natural
log).  Cases: FULL_PREFIX / VISUAL_ONLY, lse_in, d = 64 and 128, ragged seq_len,
query-row counts that leave padded 128-row blocks, key ranges spanning several
chunks with a ragged last stage, and NaN rows past seq_len (must not leak)."""
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


def _check(out, lse, ref, ref_lse, absm):
    err = np.abs(out - ref)
    bound = absm * 2.0 ** -8 + 1e-5
    worst = (err / bound).max()
    assert worst <= 1.0, f"max err / bound = {worst:.3f}, max abs err {err.max():.3e}"
    assert np.abs(lse - ref_lse).max() < 2e-4


def _run(svl, orc, wl, seed, flags=0, use_lse_in=False, poison=False):
    x = gen.make_decode_inputs(wl, seed=seed)
    if poison:  # rows past seq_len never written: NaN must not reach the output (0 * NaN)
        for b in range(wl.B):
            L = int(x["seq_len"][b])
            x["K"][b, :, L:] = float("nan")
            x["V"][b, :, L:] = float("nan")
    ref, ref_lse, absm = orc.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, flags=flags)
    dev = {k: v.cuda() for k, v in x.items()}
    lse_in = torch.as_tensor(ref_lse, dtype=torch.float32).cuda() if use_lse_in else None
    out, lse = svl.question_attention(dev["q"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, flags=flags,
                                      lse_in=lse_in)
    torch.cuda.synchronize()
    _check(out.cpu().double().numpy(), lse.cpu().double().numpy(), ref, ref_lse, absm)
    return out


@pytest.mark.parametrize("B,H,Hkv,d,vb,nv,ta,n_q,lens", [
    (1, 28, 4, 128, 32, 2048, 300, 32, None),         # NVILA-shaped: 224 rows, one padded block
    (2, 14, 2, 128, 40, 1500, 700, 37, [2240, 1999]),  # 259 rows: 3 blocks; ragged seq_len per b
    (1, 16, 2, 64, 8, 2000, 200, 8, None),             # d = 64
    (1, 4, 1, 128, 16, 1500, 600, 130, None),          # g = 4, 520 rows: 5 blocks
])
@pytest.mark.parametrize("flags", [0, 1])
def test_question_attention_shapes(svl, orc, B, H, Hkv, d, vb, nv, ta, n_q, lens, flags):
    wl = gen.DecodeWorkload("qa", B, H, Hkv, d, vb, nv, ta, 64, n_q, 256, seq_lens=lens)
    _run(svl, orc, wl, seed=21 + n_q, flags=flags)


def test_question_attention_lse_in(svl, orc):
    wl = gen.DecodeWorkload("qa", 1, 28, 4, 128, 32, 2048, 300, 64, 32, 256)
    _run(svl, orc, wl, seed=5, use_lse_in=True)


def test_question_attention_nan_past_seq_len(svl, orc):
    # capacity well past seq_len, rows there NaN; the last stage of the last chunk is ragged
    wl = gen.DecodeWorkload("qa", 2, 14, 2, 128, 32, 1800, 333, 64, 16, 256, cap=2600, seq_lens=[2165, 2101])
    _run(svl, orc, wl, seed=6, poison=True)


def test_question_attention_feeds_retrieve(svl, orc):
    # the attention pass's LSE as svl_retrieve's lse_in gives the retrieval of the
    # self-normalising path (the column-mass pass on the same normalisation)
    wl = gen.DecodeWorkload("qa", 1, 28, 4, 128, 32, 3000, 300, 300, 32, 256)
    x = gen.make_decode_inputs(wl, seed=8)
    dev = {k: v.cuda() for k, v in x.items()}
    _, lse = svl.question_attention(dev["q"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv)
    s1 = torch.empty(1, wl.Hkv, wl.nv, dtype=torch.float32, device="cuda")
    s2 = torch.empty_like(s1)
    svl.retrieve(dev["q"], dev["K"], dev["seq_len"], wl.vb, wl.nv, wl.k, scores_out=s1)
    svl.retrieve(dev["q"], dev["K"], dev["seq_len"], wl.vb, wl.nv, wl.k, lse_in=lse, scores_out=s2)
    torch.cuda.synchronize()
    a, b = s1.cpu().double().numpy(), s2.cpu().double().numpy()
    assert np.abs(a - b).max() <= 1e-4 * np.abs(a).max()


def test_question_attention_rejects(svl):
    q = torch.zeros(1, 4, 8, 128, dtype=torch.bfloat16, device="cuda")
    K = torch.zeros(1, 2, 600, 128, dtype=torch.bfloat16, device="cuda")
    V = torch.zeros(1, 2, 500, 128, dtype=torch.bfloat16, device="cuda")
    sl = torch.tensor([550], dtype=torch.int32, device="cuda")
    with pytest.raises(svl.SvlError):  # K / V capacities differ
        svl.question_attention(q, K, V, sl, 8, 400)
    with pytest.raises(svl.SvlError):  # unknown flag
        svl.question_attention(q, K, K, sl, 8, 400, flags=svl.SVL_SELECT_SHARED)
