"""Multi-GPU host logic on CPU: the (batch x KV-head)
partition covers every unit exactly once, and a world_size-2 gloo run of
the per-rank slices + the all-gather of head outputs reproduces the
single-process result bitwise (the per-unit computation -- here the fp64
oracle -- does not depend on the partition)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_17777_b200 import inputs as gen
from paper_2510_17777_b200 import sharding


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_plan_covers_units_once(P):
    B, H, Hkv = 16, 28, 4
    seen = np.zeros((B, Hkv), int)
    for r in range(P):
        sp = sharding.plan(B, H, Hkv, P, r)
        seen[sp.b0:sp.b1, sp.kv0:sp.kv1] += 1
        assert sp.H_local * sp.B_local * P == B * H
    assert (seen == 1).all()


def test_plan_rejects_indivisible_batch():
    with pytest.raises(ValueError):
        sharding.plan(1, 28, 4, 8, 0)       # B=1 cannot be split over 2 batch shards


def test_assemble_roundtrip():
    B, H, Hkv, d, P = 4, 8, 2, 16, 4
    full = torch.randn(B, H, d)
    plans = [sharding.plan(B, H, Hkv, P, r) for r in range(P)]
    parts = [full[sp.b0:sp.b1, sp.kv0 * sp.g:sp.kv1 * sp.g].contiguous() for sp in plans]
    assert torch.equal(sharding.assemble(parts, plans, B, H), full)


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
    wl = gen.DecodeWorkload("shard", 4, 8, 2, 32, 4, 300, 20, 30, 1, 64)
    x = gen.make_decode_inputs(wl, seed=5)
    sp = sharding.plan(wl.B, wl.H, wl.Hkv, world, rank)
    ql, Kl, Vl, sl = sharding.local_inputs(sp, x["q"], x["K"], x["V"], x["seq_len"])
    idx, _, _ = oracle.retrieve(ql, Kl.contiguous(), sl, wl.vb, wl.nv, wl.k)
    out, _ = oracle.sparse_decode(ql[:, 0].contiguous(), Kl.contiguous(), Vl.contiguous(), sl,
                                  wl.vb, wl.nv, idx)
    full = sharding.all_gather_heads(torch.from_numpy(out), sp, wl.H)
    if rank == 0:
        q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather_equals_single_process():
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = gen.DecodeWorkload("shard", 4, 8, 2, 32, 4, 300, 20, 30, 1, 64)
    x = gen.make_decode_inputs(wl, seed=5)
    idx, _, _ = oracle.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k)
    ref, _ = oracle.sparse_decode(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx)
    assert np.array_equal(got, ref)
