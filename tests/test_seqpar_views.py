"""Host logic of the sequence split on CPU: the shard views
cover every cache row of the attended set exactly once (system text on the
first shard, later text on the last), and with gloo world 2 the per-shard
partial decodes (fp64 oracle on each view) exchanged and merged by the a5
log-sum-exp rule reproduce the unsharded decode."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_17777_b200 import inputs as gen
from paper_2510_17777_b200 import seqpar


@pytest.mark.parametrize("P_s", [1, 2, 4, 8])
def test_views_partition_rows(P_s):
    vb, nv, cap, L = 32, 1024, 1400, 1380
    seen = np.zeros(cap, int)
    for s in range(P_s):
        v = seqpar.shard_view(vb, nv, cap, P_s, s)
        L_v = int(seqpar.view_seq_len(v, torch.tensor([L]))[0])
        assert v.vb + v.nv <= L_v <= v.rows
        rows = list(range(v.row0, v.row0 + v.vb)) + list(range(v.row0 + v.vb, v.row0 + v.vb + v.nv)) + \
            list(range(v.row0 + v.vb + v.nv, v.row0 + L_v))
        seen[rows] += 1
        assert v.lo == s * (nv // P_s) and v.row0 + v.vb == vb + v.lo
    assert (seen[:L] == 1).all() and (seen[L:] == 0).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    wl = gen.DecodeWorkload("sp", 1, 8, 2, 32, 4, 256, 20, 40, 1, 64)
    x = gen.make_decode_inputs(wl, seed=5)
    idx, _, _ = oracle.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k)
    v = seqpar.shard_view(wl.vb, wl.nv, x["K"].shape[2], world, rank)
    Kv = x["K"][:, :, v.row0:v.row0 + v.rows]
    Vv = x["V"][:, :, v.row0:v.row0 + v.rows]
    sl = seqpar.view_seq_len(v, x["seq_len"])
    loc = [[j - v.lo for j in idx[0, G] if v.lo <= j < v.lo + v.nv] for G in range(wl.Hkv)]
    n = max(len(r) for r in loc)
    # the oracle takes a dense index list: decode each KV group with its own local rows
    out = np.zeros((1, wl.H, wl.d))
    lse = np.zeros((1, wl.H))
    for G in range(wl.Hkv):
        ix = np.array([[loc[G]] * wl.Hkv], np.int32)
        o, l = oracle.sparse_decode(x["q_dec"], Kv.contiguous(), Vv.contiguous(), sl, v.vb, v.nv, ix)
        out[0, G * wl.g:(G + 1) * wl.g] = o[0, G * wl.g:(G + 1) * wl.g]
        lse[0, G * wl.g:(G + 1) * wl.g] = l[0, G * wl.g:(G + 1) * wl.g]
    _ = n
    outs = [torch.empty(1, wl.H, wl.d, dtype=torch.float64) for _ in range(world)]
    lses = [torch.empty(1, wl.H, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(outs, torch.from_numpy(out))
    dist.all_gather(lses, torch.from_numpy(lse))
    if rank == 0:
        L = torch.stack(lses)
        w = torch.softmax(L, dim=0)
        merged = (w[..., None] * torch.stack(outs)).sum(0)
        q.put((merged.numpy(), torch.logsumexp(L, dim=0).numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_split_decode_merges_to_unsharded():
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, got_lse = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = gen.DecodeWorkload("sp", 1, 8, 2, 32, 4, 256, 20, 40, 1, 64)
    x = gen.make_decode_inputs(wl, seed=5)
    idx, _, _ = oracle.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k)
    ref, ref_lse = oracle.sparse_decode(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx)
    assert np.allclose(got, ref, rtol=0, atol=1e-12) and np.allclose(got_lse, ref_lse, rtol=0, atol=1e-12)
