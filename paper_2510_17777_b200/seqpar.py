"""Sequence split (context parallel) of one request's fresh decode step
(SURVEY.md 8(f) f3 / 8(e) e4): with B = 1 there are only Hkv units, so 8 GPUs
need each unit's visual span split over P_s ranks (4 KV heads x 2 halves).

Each rank holds a view of its shard of the cache -- the system text on the
first shard, the later text (question, answer, current token) on the last --
and the fresh step runs as library calls with three exchanges between the
shards (PAPER.md:124's retrieval + decode, made sequence-parallel):

  1. svl_retrieve_partial_lse            -> exchange -> svl_lse_combine
  2. svl_retrieve(SELECT_ONLY, lse_in)   -> exchange scores -> svl_topk
                                          -> svl_shard_indices
  3. svl_sparse_decode_attn(IDX_PADDED)  -> exchange (out, lse) -> svl_merge_partials

Every step of the method runs in the library's kernels; this module only
slices views and moves tensors (torch.distributed all-gathers, or a list for
the one-GPU simulation the tests use)."""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Optional

import torch

from . import svl


@dataclasses.dataclass(frozen=True)
class ShardView:
    s: int        # shard index
    P_s: int
    row0: int     # first cache row of the view
    rows: int     # rows of the view (its capacity)
    vb: int       # visual_begin inside the view
    nv: int       # visual rows of the shard
    lo: int       # first visual index of the shard (relative to the unit's visual span)


def shard_view(vb: int, nv: int, capacity: int, P_s: int, s: int) -> ShardView:
    """Shard s of P_s of a cache with rows [0, vb) system, [vb, vb + nv) visual, [vb + nv, L)
    later text: the first shard also holds the system rows, the last one the later text."""
    if nv % P_s:
        raise ValueError(f"visual_len {nv} not divisible by P_s = {P_s}")
    nvl = nv // P_s
    lo = s * nvl
    start = 0 if s == 0 else vb + lo
    end = capacity if s == P_s - 1 else vb + lo + nvl
    return ShardView(s, P_s, start, end - start, vb if s == 0 else 0, nvl, lo)


def view_seq_len(v: ShardView, seq_len: torch.Tensor) -> torch.Tensor:
    """seq_len of the view: the shard's rows, plus the later text on the last shard."""
    if v.s == v.P_s - 1:
        return (seq_len - v.row0).to(torch.int32)
    return torch.full_like(seq_len, v.vb + v.nv, dtype=torch.int32)


class ShardState:
    """Per-shard buffers of one layer's step (kept across calls: graph-friendly)."""

    def __init__(self, q, K, V, seq_len, vb, nv, k, P_s, s, ws=None):
        B, H, d = q.shape
        self.v = shard_view(vb, nv, K.shape[2], P_s, s)
        self.q1 = q.view(B, 1, H, d)
        self.q = q
        self.K = K[:, :, self.v.row0:self.v.row0 + self.v.rows]
        self.V = V[:, :, self.v.row0:self.v.row0 + self.v.rows]
        self.seq = view_seq_len(self.v, seq_len)
        self.k = k
        self.Hkv = K.shape[1]
        self.ws = ws or svl.Workspace(q.device)
        self.ws_d = svl.Workspace(q.device)
        self.lse = torch.empty(B, 1, H, device=q.device)
        self.scores = torch.empty(B, self.Hkv, self.v.nv, device=q.device)
        self.idx_loc = torch.empty(B, self.Hkv, min(k, self.v.nv - 1), dtype=torch.int32, device=q.device)
        self.local = torch.empty(B, self.Hkv, k, dtype=torch.int32, device=q.device)
        self.out = torch.empty(B, H, d, device=q.device)
        self.lse_out = torch.empty(B, H, device=q.device)

    def phase1(self):
        svl.retrieve_partial_lse(self.q1, self.K, self.seq, self.v.vb, self.v.nv, flags=svl.SVL_SHARD_VIEW,
                                 lse_out=self.lse, ws=self.ws)
        return self.lse

    def phase2(self, lse_global):
        svl.retrieve(self.q1, self.K, self.seq, self.v.vb, self.v.nv, self.idx_loc.shape[-1],
                     flags=svl.SVL_RETRIEVE_SELECT_ONLY | svl.SVL_SHARD_VIEW, lse_in=lse_global,
                     idx_out=self.idx_loc, scores_out=self.scores, ws=self.ws)
        return self.scores

    def phase3(self, idx_global):
        svl.shard_indices(idx_global, self.v.lo, self.v.lo + self.v.nv, out=self.local)
        svl.sparse_decode_attn(self.q, self.K, self.V, self.seq, self.v.vb, self.v.nv, self.local,
                               flags=svl.SVL_IDX_PADDED, out=self.out, lse_out=self.lse_out, ws=self.ws_d)
        return self.out, self.lse_out


def combine_phase1(lse_parts: torch.Tensor) -> torch.Tensor:
    return svl.lse_combine(lse_parts)


def combine_phase2(score_parts: torch.Tensor, k: int, ws=None) -> torch.Tensor:
    """score_parts [P_s][B][Hkv][nvl] -> the unit's ascending kept indices [B][Hkv][k]."""
    P_s, B, Hkv, nvl = score_parts.shape
    full = score_parts.permute(1, 2, 0, 3).reshape(B * Hkv, P_s * nvl)
    return svl.topk(full, k, ws=ws).view(B, Hkv, k)


def simulated_step(q, K, V, seq_len, vb: int, nv: int, k: int, P_s: int):
    """All P_s shards on one device, the exchanges as stacks.  Returns (out, lse, idx)."""
    st = [ShardState(q, K, V, seq_len, vb, nv, k, P_s, s) for s in range(P_s)]
    lse = combine_phase1(torch.stack([x.phase1() for x in st]))
    idx = combine_phase2(torch.stack([x.phase2(lse) for x in st]), k)
    parts = [x.phase3(idx) for x in st]
    out, lse_o = svl.merge_partials(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]))
    return out, lse_o, idx


def distributed_step(state: ShardState, group, gather: Optional[Callable] = None):
    """One rank's fresh step; `group` = the sequence-parallel process group (size P_s).
    gather(t) -> [P_s, *t.shape] (default: torch.distributed all_gather_into_tensor)."""
    import torch.distributed as dist

    def _gather(t):
        t = t.contiguous()
        buf = t.new_empty((dist.get_world_size(group),) + tuple(t.shape))
        dist.all_gather_into_tensor(buf, t, group=group)
        return buf

    g = gather or _gather
    lse = combine_phase1(g(state.phase1()))
    idx = combine_phase2(g(state.phase2(lse)), state.k)
    out, lse_o = state.phase3(idx)
    return svl.merge_partials(g(out), g(lse_o))
