"""Seeded synthetic input generator shared by the oracle tests, the CUDA parity
tests and bench.py.

This module holds NONE of the method's arithmetic (no attention, softmax,
relevance, top-k or salience).  It only produces bf16 tensors with the shapes
and value structure of the paper's workloads:

* counter-based generator: u64_e = splitmix64(key + (e+1)*GOLDEN) with
  key = splitmix64(seed ^ fnv1a64(tag)); uniforms from the top 53 bits;
  normals by Box-Muller (one normal per two uniforms, cos branch).
* K_visual = 0.5*mu_frame + z (frames of `frame` tokens share mu; video-like
  temporal redundancy), K_text, V ~ N(0,1), q ~ 2*N(0,1) (scaled logit std ~2).
* planted structure per (b, KV group): `sinks` visual rows get a +6 mean-logit
  boost along the group's mean query direction (visual attention sinks,
  PAPER.md:160) and `needles` rows at evenly spaced depths get +4 (V-NIAH,
  PAPER.md:340-351).
* optional "gapped" variant: a random k-subset of visual rows gets +gamma
  mean-logit boost so the k / k+1 relevance gap is wide (strict index parity).

Values are generated with torch int64/float64 ops on any device.  The same
(seed, workload) gives the same bits on the same device type; CPU and GPU
log/cos may differ in the last ulp, so parity tests always copy ONE generated
tensor to both the oracle and the kernel.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import torch

_MASK64 = (1 << 64) - 1


def _s64(x: int) -> int:
    x &= _MASK64
    return x - (1 << 64) if x >= (1 << 63) else x


GOLDEN = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def fnv1a64(s: str) -> int:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h ^= ch
        h = (h * 0x100000001B3) & _MASK64
    return h


def splitmix64_py(z: int) -> int:
    """Scalar reference (pure Python ints) used to pin the tensor version."""
    z &= _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    # logical shift right on int64 (arithmetic shift, then clear sign-extension)
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def _key(tag: str, seed: int) -> int:
    return splitmix64_py((seed & _MASK64) ^ fnv1a64(tag))


def stream_u64(tag: str, seed: int, n: int, device="cpu", offset: int = 0) -> torch.Tensor:
    key = _s64(_key(tag, seed))
    e = torch.arange(offset + 1, offset + n + 1, dtype=torch.int64, device=device)
    return splitmix64(e * GOLDEN + key)


def uniform01(tag: str, seed: int, n: int, device="cpu", offset: int = 0) -> torch.Tensor:
    u = stream_u64(tag, seed, n, device, offset)
    return (_lsr(u, 11).to(torch.float64) + 0.5) * (2.0 ** -53)


def normal(tag: str, seed: int, n: int, device="cpu") -> torch.Tensor:
    """n standard normals; element e uses uniforms 2e, 2e+1 of the stream."""
    out = torch.empty(n, dtype=torch.float64, device=device)
    chunk = 1 << 24
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        u = uniform01(tag, seed, 2 * m, device, offset=2 * s).view(m, 2)
        out[s:s + m] = torch.sqrt(-2.0 * torch.log(u[:, 0])) * torch.cos((2.0 * math.pi) * u[:, 1])
    return out


def to_bf16(x: torch.Tensor) -> torch.Tensor:
    """float64 -> float32 (RNE) -> bfloat16 (RNE)."""
    return x.to(torch.float32).to(torch.bfloat16)


def randint_perm(tag: str, seed: int, n: int, device="cpu") -> torch.Tensor:
    """A seeded permutation of range(n) (argsort of uniform keys, stable)."""
    u = uniform01(tag, seed, n, device)
    return torch.argsort(u, stable=True)


# --------------------------------------------------------------------------
# Decode-stage workload (retrieve + sparse decode attention)
# --------------------------------------------------------------------------


@dataclasses.dataclass
class DecodeWorkload:
    """One decoder layer's KV cache + the query rows for one step.

    Sequence layout per batch row b (reading A20):
      [0, vb)            system text rows
      [vb, vb+nv)        visual rows (after prefill pruning)
      [vb+nv, seq_len)   question / answer / generated rows, current token last
    """

    name: str = "toy"
    B: int = 1
    H: int = 4
    Hkv: int = 2
    d: int = 64
    vb: int = 8
    nv: int = 512
    t_after: int = 24          # text rows after the visual span (incl. current token)
    k: int = 64
    n_q: int = 1
    frame: int = 256
    sinks: int = 8
    needles: int = 5
    gap_gamma: float = 0.0     # >0: gapped variant (random k-subset boosted)
    cap: Optional[int] = None  # capacity rows (>= seq_len); default seq_len + 16
    seq_lens: Optional[list] = None  # per-b override of seq_len (ragged text)

    @property
    def g(self) -> int:
        return self.H // self.Hkv

    @property
    def seq_len(self) -> int:
        return self.vb + self.nv + self.t_after

    @property
    def capacity(self) -> int:
        if self.cap is not None:
            return self.cap
        m = max(self.seq_lens) if self.seq_lens else self.seq_len
        return m + 16


# The five BASELINE.json configs.  vb = 32 system rows
# except toy (8); the remainder of the text follows the visual span.
CONFIGS = {
    "toy": DecodeWorkload("toy", 1, 4, 2, 64, 8, 512, 24, 64, 1, 256),
    "nvila-4k": DecodeWorkload("nvila-4k", 1, 28, 4, 128, 32, 4096, 96, 1024, 1, 4096),
    "long-video": DecodeWorkload("long-video", 1, 28, 4, 128, 32, 32768, 480 + 256, 3277, 1, 256),
    "multi-turn": DecodeWorkload("multi-turn", 8, 28, 4, 128, 32, 16384, 32 + 250, 1638, 1, 256),
    "sweep": DecodeWorkload("sweep", 16, 28, 4, 128, 32, 65536, 480 + 256, 6554, 1, 256),
}


def make_decode_inputs(wl: DecodeWorkload, seed: int = 0, device="cpu") -> dict:
    """Returns bf16 tensors: q [B][n_q][H][d], K/V [B][Hkv][cap][d], and int32
    seq_len [B].  q_dec = q[:, n_q-1] is the decode query of the step."""
    B, H, Hkv, d, g = wl.B, wl.H, wl.Hkv, wl.d, wl.g
    cap = wl.capacity
    tag = f"{wl.name}/B{B}H{H}K{Hkv}d{d}nv{wl.nv}vb{wl.vb}cap{cap}"
    q = 2.0 * normal(tag + "/q", seed, B * wl.n_q * H * d, device).view(B, wl.n_q, H, d)
    q = to_bf16(q)
    K = normal(tag + "/K", seed, B * Hkv * cap * d, device).view(B, Hkv, cap, d)
    V = to_bf16(normal(tag + "/V", seed, B * Hkv * cap * d, device).view(B, Hkv, cap, d))
    nf = (wl.nv + wl.frame - 1) // wl.frame
    mu = normal(tag + "/mu", seed, B * Hkv * nf * d, device).view(B, Hkv, nf, d)
    fr = torch.arange(wl.nv, device=device) // wl.frame
    K[:, :, wl.vb:wl.vb + wl.nv, :] += 0.5 * mu[:, :, fr, :]

    # Planted structure along each group's mean query direction u_G, scaled so
    # the mean scaled logit over the group's heads rises by beta.
    qf = q.to(torch.float64)                                      # [B][nq][H][d]
    qg = qf[:, -1].reshape(B, Hkv, g, d)
    u = qg.sum(2)
    u = u / u.norm(dim=-1, keepdim=True).clamp_min(1e-30)         # [B][Hkv][d]
    proj = (qg * u[:, :, None, :]).sum(-1).mean(-1)               # [B][Hkv]
    unit = math.sqrt(d) / proj.abs().clamp_min(1e-6)              # K offset per +1 logit

    def boost(rows: torch.Tensor, beta: float):
        # rows: [B][Hkv][m] visual indices
        for b in range(B):
            for G in range(Hkv):
                r = rows[b, G] + wl.vb
                K[b, G, r, :] += (beta * unit[b, G]) * u[b, G]

    if wl.sinks > 0 and wl.nv >= wl.sinks:
        sink_rows = torch.stack([
            torch.stack([randint_perm(f"{tag}/sink/{b}/{G}", seed, wl.nv, device)[:wl.sinks]
                         for G in range(Hkv)]) for b in range(B)])
        boost(sink_rows, 6.0)
    if wl.needles > 0 and wl.nv >= wl.needles:
        depth = torch.tensor([int((2 * i + 1) * wl.nv / (2 * wl.needles)) for i in range(wl.needles)],
                             device=device)
        boost(depth.expand(B, Hkv, -1), 4.0)
    if wl.gap_gamma > 0 and 0 < wl.k < wl.nv:
        sub = torch.stack([
            torch.stack([randint_perm(f"{tag}/gap/{b}/{G}", seed, wl.nv, device)[:wl.k]
                         for G in range(Hkv)]) for b in range(B)])
        boost(sub, wl.gap_gamma)
    K = to_bf16(K)

    if wl.seq_lens is not None:
        seq = torch.tensor(wl.seq_lens, dtype=torch.int32, device=device)
    else:
        seq = torch.full((B,), wl.seq_len, dtype=torch.int32, device=device)
    return {"q": q.contiguous(), "q_dec": q[:, -1].contiguous(), "K": K.contiguous(),
            "V": V.contiguous(), "seq_len": seq}


# --------------------------------------------------------------------------
# Prefill workload (vision-encoder salience + per-frame prune)
# --------------------------------------------------------------------------


@dataclasses.dataclass
class PrefillWorkload:
    name: str = "prune"
    F: int = 256          # frames
    S: int = 0            # summary rows per frame (0 = SigLIP-style, INTRA_VISUAL)
    Nf: int = 512         # visual tokens per frame
    He: int = 16          # encoder heads
    de: int = 72          # encoder head dim
    sparsity: float = 0.75


def make_prefill_inputs(wl: PrefillWorkload, seed: int = 0, device="cpu") -> dict:
    """Qe, Ke bf16 [F][S+Nf][He][de] with token clusters (objects) so
    attention has structure; std chosen so logits have std ~1.5."""
    n = wl.F * (wl.S + wl.Nf) * wl.He * wl.de
    tag = f"{wl.name}/F{wl.F}S{wl.S}N{wl.Nf}H{wl.He}d{wl.de}"
    shape = (wl.F, wl.S + wl.Nf, wl.He, wl.de)
    base = normal(tag + "/c", seed, wl.F * 16 * wl.He * wl.de, device).view(wl.F, 16, wl.He, wl.de)
    cl = (torch.arange(wl.S + wl.Nf, device=device) * 7) % 16
    Q = normal(tag + "/Q", seed, n, device).view(shape) + 0.7 * base[:, cl]
    Kt = normal(tag + "/K", seed, n, device).view(shape) + 0.7 * base[:, cl]
    s = math.sqrt(1.5) / (1.0 + 0.49) ** 0.5
    return {"Qe": to_bf16(s * Q).contiguous(), "Ke": to_bf16(s * Kt).contiguous()}


def make_saliency(B: int, N: int, seed: int = 0, ties: bool = False, device="cpu") -> torch.Tensor:
    """fp32 saliency [B][N] (positive, heavy-tailed); `ties` quantises values
    so many exact ties exist (tie-break tests)."""
    z = normal(f"sal/B{B}N{N}", seed, B * N, device).view(B, N)
    x = torch.exp(1.5 * z) / N
    if ties:
        x = torch.round(x * N * 4) / (N * 4)
    return x.to(torch.float32).contiguous()
