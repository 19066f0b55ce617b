"""svl_sparse_decode_attn's split-K decomposition (SURVEY.md 8(a) a4 + a5): the
attended rows of each (b, KV group) unit are cut into S splits, one CTA each,
merged after a grid-wide barrier.  The result must match the fp64 oracle for
any S (pinned with SVL_PIN_SPLITS), including more splits than rows (empty
partials), one split (no merge), and every split count reruns bitwise; the
barrier's self-resetting counters must survive back-to-back calls with
different split counts on one workspace, inside a CUDA graph too."""
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


def _case(orc, name, seed):
    wl = gen.CONFIGS[name]
    cpu = gen.make_decode_inputs(wl, seed=seed)
    oi, _, _ = orc.retrieve(cpu["q"], cpu["K"], cpu["seq_len"], wl.vb, wl.nv, wl.k, nthreads=NTH)
    oo, ol = orc.sparse_decode(cpu["q_dec"], cpu["K"], cpu["V"], cpu["seq_len"], wl.vb, wl.nv, oi,
                               nthreads=NTH)
    dev = {kk: v.cuda() for kk, v in cpu.items()}
    return wl, dev, torch.as_tensor(oi).cuda(), oo, ol


@pytest.mark.parametrize("name,splits", [("toy", [1, 2, 7, 16, 74]),
                                         ("long-video", [1, 3, 8, 16, 37])])
def test_decode_any_split_count_matches_oracle(svl, orc, name, splits):
    wl, dev, idx, oo, ol = _case(orc, name, seed=81)
    ws = svl.Workspace()
    for S in splits:
        # S <= 16: the cluster (DSMEM) merge by default, and the grid (L2) merge forced
        for extra in ((0, svl.SVL_DECODE_GRID_MERGE) if 1 < S <= 16 else (0,)):
            fl = svl.SVL_PIN_SPLITS(S) | extra
            lse = torch.empty(wl.B, wl.H, device="cuda")
            a, _ = svl.sparse_decode_attn(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, idx,
                                          flags=fl, lse_out=lse, ws=ws)
            a, lse_a = a.clone(), lse.clone()
            # the rerun with SVL_DECODE_STATIC_PREFIX (prompt rows gathered before the PDL wait)
            b, _ = svl.sparse_decode_attn(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, idx,
                                          flags=fl | svl.SVL_DECODE_STATIC_PREFIX, lse_out=lse, ws=ws)
            torch.cuda.synchronize()
            assert torch.equal(a, b) and torch.equal(lse_a, lse), f"S={S} not bitwise repeatable"
            mx, rel = parity.check_attention(a.cpu().numpy(), lse_a.cpu().numpy(), oo, ol)
            print(f"{name} S={S} flags={fl:#x}: max-abs {mx:.2e} rel {rel:.2e}")
    assert ws.flags() == 0
    # the header counters are back to zero after every call
    assert int(ws.buf[12:16].view(torch.int32).abs().sum()) == 0  # the push counter (header word 3)


def test_decode_planner_default_and_graph_replay(svl, orc):
    """The planner's split count, inside a CUDA graph replayed many times (the bench's
    arrangement: PDL between consecutive layers) -- results equal the eager call."""
    wl, dev, idx, oo, ol = _case(orc, "long-video", seed=82)
    ws = svl.Workspace()
    ref, _ = svl.sparse_decode_attn(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, idx, ws=ws)
    ref = ref.clone()
    parity.check_attention(ref.cpu().numpy(), None, oo, ol)
    outs = [torch.empty_like(ref) for _ in range(6)]

    def body():  # alternating with / without SVL_DECODE_STATIC_PREFIX (idx is not written here)
        for i, o in enumerate(outs):
            svl.sparse_decode_attn(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, idx,
                                   flags=svl.SVL_DECODE_STATIC_PREFIX if i % 2 else 0, out=o, ws=ws)
    body()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            body()
    for _ in range(50):
        g.replay()
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    assert ws.flags() == 0


def test_decode_pin_too_many_splits_rejected(svl):
    wl = gen.CONFIGS["multi-turn"]  # 32 units: 32 * 255 CTAs cannot be co-resident
    x = gen.make_decode_inputs(gen.DecodeWorkload(**{**wl.__dict__, "nv": 2048, "k": 200}), seed=83,
                               device="cuda")
    idx = torch.arange(200, dtype=torch.int32, device="cuda").expand(wl.B, wl.Hkv, 200).contiguous()
    with pytest.raises(svl.SvlError) as e:
        svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, 2048, idx,
                               flags=svl.SVL_PIN_SPLITS(255))
    assert e.value.status == 5  # SVL_ERR_UNSUPPORTED


@pytest.mark.parametrize("B", [2, 3, 4, 6])
def test_decode_planner_batch_sweep_matches_oracle(svl, orc, B):
    """Planner defaults at B*Hkv = 8..24 units: where the S-CTA clusters are not all
    co-resident the planner narrows the cluster or switches to the L2 merge (api.cu
    plan_decode); whichever path runs must match the oracle and rerun bitwise."""
    base = gen.CONFIGS["long-video"]
    wl = gen.DecodeWorkload(**{**base.__dict__, "name": f"lvB{B}", "B": B, "nv": 4096, "k": 1024,
                               "seq_lens": None})
    cpu = gen.make_decode_inputs(wl, seed=90 + B)
    g = torch.Generator().manual_seed(B)
    oi = torch.stack([torch.stack([torch.sort(torch.randperm(wl.nv, generator=g)[:wl.k])[0]
                                   for _ in range(wl.Hkv)]) for _ in range(B)]).to(torch.int32).numpy()
    oo, ol = orc.sparse_decode(cpu["q_dec"], cpu["K"], cpu["V"], cpu["seq_len"], wl.vb, wl.nv, oi, nthreads=NTH)
    dev = {kk: v.cuda() for kk, v in cpu.items()}
    idx = torch.as_tensor(oi).cuda()
    ws = svl.Workspace()
    lse = torch.empty(wl.B, wl.H, device="cuda")
    a, _ = svl.sparse_decode_attn(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, idx,
                                  lse_out=lse, ws=ws)
    a, lse_a = a.clone(), lse.clone()
    b, _ = svl.sparse_decode_attn(dev["q_dec"], dev["K"], dev["V"], dev["seq_len"], wl.vb, wl.nv, idx,
                                  flags=svl.SVL_DECODE_STATIC_PREFIX, lse_out=lse, ws=ws)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(lse_a, lse)
    parity.check_attention(a.cpu().numpy(), lse_a.cpu().numpy(), oo, ol)
    assert ws.flags() == 0


@pytest.mark.parametrize("name,up", [("toy", "fresh"), ("nvila-4k", "fresh"), ("long-video", "decode")])
def test_decode_early_gathers_under_a_racing_seq_len_writer(svl, name, up):
    """SVL_DECODE_STATIC_PREFIX reads seq_len speculatively before the PDL wait and checks it
    after the batch loop.  Here the upstream kernel (a fused fresh step or a plain decode, a PDL
    primary) writes its fp32 output over the very words the decode then reads as seq_len, in a
    CUDA graph (eager launches leave CPU gaps: nothing would race): the early read sees the old
    value, the checked read the upstream's bits (clamped to the span, device flag raised), so
    every replay takes the miss path (a build that flags misses counted 50 of 50:
    profiles/specmiss_r03.txt).  The result must equal a plain call on the final value."""
    wl = gen.CONFIGS[name]
    x = gen.make_decode_inputs(wl, seed=95, device="cuda")
    idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k).clone()
    buf = torch.zeros(wl.B, wl.H, wl.d, device="cuda")  # the upstream's out
    seq_view = buf.view(-1).view(torch.int32)[:wl.B]    # ... whose first words are the seq_len
    ws_u, ws_d, ws_r = svl.Workspace(), svl.Workspace(), svl.Workspace()
    a = torch.empty(wl.B, wl.H, wl.d, device="cuda")

    def body():
        seq_view.copy_(x["seq_len"])
        if up == "fresh":
            svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, out=buf, ws=ws_u)
        else:
            svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx, out=buf, ws=ws_u)
        svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], seq_view, wl.vb, wl.nv, idx,
                               flags=svl.SVL_DECODE_STATIC_PREFIX, out=a, ws=ws_d)
    body()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            body()
    for it in range(20):
        g.replay()
        torch.cuda.synchronize()
        ref, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], seq_view, wl.vb, wl.nv, idx, ws=ws_r)
        assert torch.equal(a, ref), f"replay {it}"
