"""Multi-GPU partitioning of the decode-stage hot path.

The unit (b, KV group G) is independent through retrieve + sparse decode
(per-group selection, reading A4), so ranks own disjoint blocks of units and
only their units' KV (a sharded cache, no replication).  The one exchange is
the all-gather of the per-head attention outputs that the next layer's
output projection needs (north star: "NCCL all-gather of head outputs").

Partition: P = P_b * P_h with P_h = gcd(P, Hkv) ranks
splitting the KV heads and P_b = P / P_h splitting the batch; rank p owns KV
heads [h0, h1) = [(p % P_h) * Hkv/P_h, ...) of batch rows
[(p // P_h) * B/P_b, ...).  Hkv = 4: P in {1, 2, 4} shard heads only; P = 8
shards heads x batch halves (needs B >= 2).
"""
from __future__ import annotations

import dataclasses
import math

import torch


@dataclasses.dataclass(frozen=True)
class ShardPlan:
    P: int
    rank: int
    B: int
    Hkv: int
    g: int
    P_b: int
    P_h: int
    b0: int
    b1: int
    kv0: int
    kv1: int

    @property
    def H_local(self) -> int:
        return (self.kv1 - self.kv0) * self.g

    @property
    def B_local(self) -> int:
        return self.b1 - self.b0


def plan(B: int, H: int, Hkv: int, P: int, rank: int) -> ShardPlan:
    if H % Hkv:
        raise ValueError("H % Hkv != 0")
    if not 0 <= rank < P:
        raise ValueError("rank outside [0, P)")
    P_h = math.gcd(P, Hkv)
    P_b = P // P_h
    if B % P_b:
        raise ValueError(f"batch {B} not divisible by the {P_b} batch shards of P={P}, Hkv={Hkv}")
    ph, pb = rank % P_h, rank // P_h
    kv_per, b_per = Hkv // P_h, B // P_b
    return ShardPlan(P, rank, B, Hkv, H // Hkv, P_b, P_h, pb * b_per, (pb + 1) * b_per,
                     ph * kv_per, (ph + 1) * kv_per)


def local_inputs(sp: ShardPlan, q: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
                 seq_len: torch.Tensor):
    """Views of this rank's slice (no copies of K/V; q made contiguous).
    q: [B][H][d] (decode) or [B][n_q][H][d]; K, V: [B][Hkv][cap][d]."""
    h0, h1 = sp.kv0 * sp.g, sp.kv1 * sp.g
    if q.dim() == 3:
        ql = q[sp.b0:sp.b1, h0:h1].contiguous()
    else:
        ql = q[sp.b0:sp.b1, :, h0:h1].contiguous()
    return (ql, K[sp.b0:sp.b1, sp.kv0:sp.kv1], V[sp.b0:sp.b1, sp.kv0:sp.kv1],
            seq_len[sp.b0:sp.b1].contiguous())


def assemble(parts: list, plans: list, B: int, H: int, d: int = None) -> torch.Tensor:
    """Place each rank's [B_local][H_local][d] block (any shape of that size)
    into [B][H][d]."""
    d = parts[0].shape[-1] if d is None else d
    out = parts[0].new_empty(B, H, d)
    for part, sp in zip(parts, plans):
        out[sp.b0:sp.b1, sp.kv0 * sp.g:sp.kv1 * sp.g] = part.view(sp.B_local, sp.H_local, d)
    return out


def all_gather_heads(out_local: torch.Tensor, sp: ShardPlan, H: int, group=None) -> torch.Tensor:
    """The per-layer exchange: all-gather every rank's [B_local][H_local][d]
    output block (equal sizes for every rank) and permute into [B][H][d]."""
    import torch.distributed as dist
    flat = out_local.contiguous().view(-1)
    gathered = flat.new_empty(sp.P * flat.numel())
    try:
        dist.all_gather_into_tensor(gathered, flat, group=group)
        parts = list(gathered.view(sp.P, -1))
    except (RuntimeError, NotImplementedError, ValueError):  # backends without the fused op
        parts = [torch.empty_like(flat) for _ in range(sp.P)]
        dist.all_gather(parts, flat, group=group)
    plans = [plan(sp.B, H, sp.Hkv, sp.P, r) for r in range(sp.P)]
    return assemble(parts, plans, sp.B, H, out_local.shape[-1])
