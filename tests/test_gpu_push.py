"""svl_sparse_decode_attn_push + svl_wait_flags (SURVEY.md 8(b) b7, 8(e) e3 fused
variant): P simulated ranks on one GPU (their "peer" buffers are all device
memory, reached through the same unified-address stores the kernel issues
over NVLink).  Every rank's gathered output must equal the unsharded decode
bitwise (per-unit split counts are pinned by the plan: same cluster size),
and every flag row must carry the epoch."""
import pytest
import torch

from paper_2510_17777_b200 import inputs as gen
from paper_2510_17777_b200 import sharding

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def svl():
    from paper_2510_17777_b200 import build, svl as mod
    build.build()
    mod.lib()
    return mod


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_push_gather_equals_unsharded(svl, P):
    # per-unit split count pinned: the planner sizes the splits by the
    # number of units, which differs between a shard and the whole batch
    pin = svl.SVL_PIN_SPLITS(8)
    wl = gen.DecodeWorkload("push", 4, 28, 4, 128, 32, 8192, 300, 819, 1, 256)
    x = gen.make_decode_inputs(wl, seed=41, device="cuda")
    idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k).clone()
    ref, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx, flags=pin)
    ref = ref.clone()
    outs = [torch.full((wl.B, wl.H, wl.d), float("nan"), device="cuda") for _ in range(P)]
    flags = [torch.zeros(P, dtype=torch.int32, device="cuda") for _ in range(P)]
    wss = [svl.Workspace() for _ in range(P)]
    plans = [sharding.plan(wl.B, wl.H, wl.Hkv, P, r) for r in range(P)]
    for epoch in (1, 2, 3):
        for o in outs:
            o.fill_(float("nan"))
        for r, sp in enumerate(plans):
            ql, Kl, Vl, sl = sharding.local_inputs(sp, x["q_dec"], x["K"], x["V"], x["seq_len"])
            il = idx[sp.b0:sp.b1, sp.kv0:sp.kv1].contiguous()
            svl.sparse_decode_attn_push(ql, Kl, Vl, sl, wl.vb, wl.nv, il, outs, flags, r, epoch,
                                        sp.b0, sp.kv0 * sp.g, flags=pin, ws=wss[r])
        for r in range(P):
            svl.wait_flags(flags[r], epoch, ws=wss[r])
        torch.cuda.synchronize()
        for r in range(P):
            assert torch.equal(outs[r], ref), f"rank {r} gathered output != unsharded (epoch {epoch})"
            assert (flags[r] == epoch).all()
            assert wss[r].flags() & svl.SVL_DEVFLAG_WAIT_TIMEOUT == 0


def test_wait_flags_timeout_is_bounded(svl):
    """A flag that never arrives sets SVL_DEVFLAG_WAIT_TIMEOUT instead of hanging."""
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    ws = svl.Workspace()
    ws.get(1024)
    ws.reset_flags()
    svl.wait_flags(flags, 5, ws=ws)
    torch.cuda.synchronize()
    assert ws.flags() & svl.SVL_DEVFLAG_WAIT_TIMEOUT
