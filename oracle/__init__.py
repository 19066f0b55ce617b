"""ctypes front-end of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2510_17777_b200) never imports this module, and this module never
imports the product package.

Every function takes CPU torch tensors (bf16 / int32 / float32) as produced by
paper_2510_17777_b200.inputs and returns float64 / int32 numpy arrays.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

VISUAL_ONLY = 1
SHARED = 2
SAL_SUMMARY, SAL_MULTI_SUMMARY, SAL_INTRA_VISUAL = 0, 1, 2

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (IEEE semantics: no fast-math, no FMA
    contraction).  Building the checker is not using it."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
                               "-ffp-contract=off", "-fno-fast-math", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P, I, I64, D, U = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double,
                           ctypes.c_uint)
        L.o_keep_budget.restype = ctypes.c_int64
        L.o_keep_budget.argtypes = [I64, D]
        L.o_retrieve.restype = I
        L.o_retrieve.argtypes = [P, I, I, I, I, I, P, I64, I64, I64, I, I, P, P, I, D, U,
                                 P, P, P, I]
        L.o_sparse_decode.restype = I
        L.o_sparse_decode.argtypes = [P, I, I, I, I, P, I64, I64, I64, P, I64, I64, I64,
                                      I, I, P, P, I, U, D, P, P, I]
        L.o_dense_attn.restype = I
        L.o_dense_attn.argtypes = [P, I, I, I, I, P, I64, I64, I64, P, I64, I64, I64, P, D,
                                   P, P, I]
        L.o_salience.restype = I
        L.o_salience.argtypes = [P, P, I, I, I, I, I, I, D, P, I]
        L.o_prune.restype = I
        L.o_prune.argtypes = [P, I, I, P, I, D, P, I, P]
        L.o_rope_remap.argtypes = [P, I, I, I, I, P, I, I, P, I, D, P, I, P]
        L.o_mrope_plan.restype = I
        L.o_mrope_plan.argtypes = [P, I, I, I, P, I, P, P]
        L.o_mrope_remap.restype = I
        L.o_mrope_remap.argtypes = [P, I, I, I, I, P, I, I, P, I, P, P, P, D, P, I, P]
        L.o_page_summary.restype = I
        L.o_page_summary.argtypes = [P, I, I, I, I64, I64, I64, I, I, I, P, P]
        L.o_retrieve_pages.restype = I
        L.o_retrieve_pages.argtypes = [P, I, I, I, I, I, P, P, I, I, D, P, P, P]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc != 0:
        raise OracleError(f"{what} failed with code {rc}")


def _u16(t: torch.Tensor) -> np.ndarray:
    assert t.dtype == torch.bfloat16 and t.device.type == "cpu"
    return t.view(torch.int16).numpy().view(np.uint16)


def _kv(t: torch.Tensor):
    """[B][Hkv][cap][d] bf16 view with contiguous last dim -> (array, strides)."""
    assert t.dim() == 4 and t.stride(3) == 1 and t.dtype == torch.bfloat16
    n = t.untyped_storage().nbytes() // 2
    whole = torch.empty(0, dtype=torch.bfloat16).set_(t.untyped_storage(), 0, (n,), (1,))
    return _u16(whole), t.storage_offset(), t.stride(0), t.stride(1), t.stride(2)


def _ptr(a: np.ndarray, off: int = 0) -> int:
    return a.ctypes.data + off * a.itemsize


def keep_budget(n: int, s: float) -> int:
    return int(lib().o_keep_budget(n, s))


def retrieve(q, K, seq_len, vb: int, nv: int, k: int, scale: float | None = None,
             flags: int = 0, lse_in=None, nthreads: int = 1):
    """Returns (idx [B][U][k] int32, scores [B][U][nv] f64, rel_gap [B][U] f64)."""
    B, n_q, H, d = q.shape
    Hkv = K.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    U = 1 if flags & SHARED else Hkv
    qa = _u16(q.contiguous())
    ka, koff, sb, sh, st = _kv(K)
    sl = seq_len.to(torch.int32).contiguous().numpy()
    idx = np.zeros((B, U, k), np.int32)
    sc = np.zeros((B, U, nv), np.float64)
    gap = np.zeros((B, U), np.float64)
    li = None
    if lse_in is not None:
        li = np.ascontiguousarray(np.asarray(lse_in, dtype=np.float64).reshape(B, n_q, H))
    rc = lib().o_retrieve(_ptr(qa), B, n_q, H, Hkv, d, _ptr(ka, koff), sb, sh, st, vb, nv,
                          _ptr(sl), _ptr(li) if li is not None else None, k, scale, flags,
                          _ptr(idx), _ptr(sc), _ptr(gap), nthreads)
    _check(rc, "o_retrieve")
    return idx, sc, gap


def sparse_decode(q, K, V, seq_len, vb: int, nv: int, idx, scale: float | None = None,
                  flags: int = 0, nthreads: int = 1):
    """q [B][H][d]; idx [B][U][k] int32 (ascending).  Returns (out [B][H][d], lse [B][H])."""
    B, H, d = q.shape
    Hkv = K.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    qa = _u16(q.contiguous())
    ka, koff, ksb, ksh, kst = _kv(K)
    va, voff, vsb, vsh, vst = _kv(V)
    sl = seq_len.to(torch.int32).contiguous().numpy()
    ix = np.ascontiguousarray(np.asarray(idx, dtype=np.int32))
    k = ix.shape[-1]
    out = np.zeros((B, H, d), np.float64)
    lse = np.zeros((B, H), np.float64)
    rc = lib().o_sparse_decode(_ptr(qa), B, H, Hkv, d, _ptr(ka, koff), ksb, ksh, kst,
                               _ptr(va, voff), vsb, vsh, vst, vb, nv, _ptr(sl), _ptr(ix), k,
                               flags, scale, _ptr(out), _ptr(lse), nthreads)
    _check(rc, "o_sparse_decode")
    return out, lse


def dense_attn(q, K, V, seq_len, scale: float | None = None, nthreads: int = 1):
    B, H, d = q.shape
    Hkv = K.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    qa = _u16(q.contiguous())
    ka, koff, ksb, ksh, kst = _kv(K)
    va, voff, vsb, vsh, vst = _kv(V)
    sl = seq_len.to(torch.int32).contiguous().numpy()
    out = np.zeros((B, H, d), np.float64)
    lse = np.zeros((B, H), np.float64)
    rc = lib().o_dense_attn(_ptr(qa), B, H, Hkv, d, _ptr(ka, koff), ksb, ksh, kst,
                            _ptr(va, voff), vsb, vsh, vst, _ptr(sl), scale, _ptr(out),
                            _ptr(lse), nthreads)
    _check(rc, "o_dense_attn")
    return out, lse


def salience(Qe, Ke, S: int, mode: int, scale: float | None = None, nthreads: int = 1):
    """Qe, Ke bf16 [F][S+Nf][He][de] -> saliency [F][Nf] (float64)."""
    F, T, He, de = Qe.shape
    Nf = T - S
    if scale is None:
        scale = 1.0 / math.sqrt(de)
    qa = _u16(Qe.contiguous())
    ka = _u16(Ke.contiguous())
    sal = np.zeros((F, Nf), np.float64)
    rc = lib().o_salience(_ptr(qa), _ptr(ka), F, S, Nf, He, de, mode, scale, _ptr(sal), nthreads)
    _check(rc, "o_salience")
    return sal


def prune(saliency, s: float, frame_offsets=None):
    """saliency fp32 [B][N] -> (kept [B][total] int32, total)."""
    sal = np.ascontiguousarray(np.asarray(saliency, dtype=np.float32))
    B, N = sal.shape
    if frame_offsets is not None:
        fo = np.ascontiguousarray(np.asarray(frame_offsets, dtype=np.int32))
        nf = len(fo) - 1
        cap = sum(max(keep_budget(int(fo[i + 1] - fo[i]), s), 0) for i in range(nf))
    else:
        fo, nf = None, 1
        cap = keep_budget(N, s)
    cap = max(cap, 1)
    kept = np.zeros((B, cap), np.int32)
    tot = ctypes.c_int32(0)
    rc = lib().o_prune(_ptr(sal), B, N, _ptr(fo) if fo is not None else None, nf, s,
                       _ptr(kept), cap, ctypes.addressof(tot))
    _check(rc, "o_prune")
    return kept[:, :tot.value], tot.value


def rope_remap(K_pre, seq_len, vb: int, nv: int, kept, base: float, cap_out: int | None = None):
    """Unified RoPE remap after pruning.  K_pre bf16 [B][Hkv][cap][d]
    (pre-RoPE keys at their original rows); kept int32 [B][k] ascending, relative to vb.
    Returns (K_post float64 [B][Hkv][cap_out][d] unrounded, rows int32 [B][cap_out] old row or -1)."""
    Kc = K_pre.contiguous()
    B, Hkv, cap, d = Kc.shape
    kp = np.ascontiguousarray(np.asarray(kept, dtype=np.int32))
    k = kp.shape[-1]
    sl = np.ascontiguousarray(np.asarray(seq_len, dtype=np.int32))
    cap_out = cap - nv + k if cap_out is None else cap_out
    out = np.zeros((B, Hkv, cap_out, d), np.float64)
    rows = np.zeros((B, cap_out), np.int32)
    ku = _u16(Kc)
    rc = lib().o_rope_remap(_ptr(ku), B, Hkv, d, cap, _ptr(sl), vb, nv, _ptr(kp), k, base, _ptr(out),
                            cap_out, _ptr(rows))
    _check(rc, "o_rope_remap")
    return out, rows


def page_summary(K, vb: int, nv: int, page: int):
    """Per-page elementwise max / min of the visual keys.
    K bf16 [B][Hkv][cap][d].  Returns (kmax, kmin) float64 [B][Hkv][nv/page][d]."""
    B, Hkv, _, d = K.shape
    ka, koff, sb, sh, st = _kv(K)
    npg = nv // page
    kmax = np.zeros((B, Hkv, npg, d), np.float64)
    kmin = np.zeros((B, Hkv, npg, d), np.float64)
    rc = lib().o_page_summary(_ptr(ka, koff), B, Hkv, d, sb, sh, st, vb, nv, page, _ptr(kmax), _ptr(kmin))
    _check(rc, "o_page_summary")
    return kmax, kmin


def retrieve_pages(q, kmax, kmin, k_pages: int, scale: float | None = None):
    """Quest-style page retrieval (reading A22).  q bf16 [B][n_q][H][d]; kmax / kmin
    float64 [B][Hkv][np][d].  Returns (page_idx [B][Hkv][k_pages] int32, scores
    [B][Hkv][np] f64, rel_gap [B][Hkv])."""
    B, n_q, H, d = q.shape
    _, Hkv, npg, _ = kmax.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    qa = _u16(q.contiguous())
    mx = np.ascontiguousarray(kmax, dtype=np.float64)
    mn = np.ascontiguousarray(kmin, dtype=np.float64)
    idx = np.zeros((B, Hkv, k_pages), np.int32)
    sc = np.zeros((B, Hkv, npg), np.float64)
    gap = np.zeros((B, Hkv), np.float64)
    rc = lib().o_retrieve_pages(_ptr(qa), B, n_q, H, Hkv, d, _ptr(mx), _ptr(mn), npg, k_pages, scale,
                                _ptr(idx), _ptr(sc), _ptr(gap))
    _check(rc, "o_retrieve_pages")
    return idx, sc, gap


def question_attention(q, K, V, seq_len, vb: int, nv: int, scale: float | None = None, flags: int = 0,
                       lse_in=None):
    """The question chunk's attention output: PAPER.md:124 runs the
    query-aware retrieval "concurrently with the FlashAttention2 path during prefill";
    this is that path's product for the n_q question rows (the last n_q rows of seq_len[b]),
    written from the definition of softmax attention, in float64 numpy:
        s[r,h,j] = scale * q[b,r,h,:] . K[b,G,j,:],  G = h // g,
                   j in the causal prefix j <= seq_len - n_q + r
                   (the visual rows [vb, vb+nv) only with VISUAL_ONLY),
        LSE[r,h] = lse_in[b,r,h] if given else log sum_j exp(s[r,h,j]),
        out[r,h] = sum_j exp(s[r,h,j] - LSE[r,h]) V[b,G,j,:].
    Returns (out [B][n_q][H][d], lse [B][n_q][H], absmass [B][n_q][H][d] =
    sum_j exp(s - LSE) |V_j| -- the scale of the rounding bound on out, reading A24)."""
    B, n_q, H, d = q.shape
    Hkv = K.shape[1]
    g = H // Hkv
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    qd = q.to(torch.float64).numpy()
    Kd = K.to(torch.float64).numpy()
    Vd = V.to(torch.float64).numpy()
    sl = seq_len.to(torch.int64).numpy()
    li = None if lse_in is None else np.asarray(lse_in, dtype=np.float64).reshape(B, n_q, H)
    out = np.zeros((B, n_q, H, d))
    lse = np.zeros((B, n_q, H))
    absmass = np.zeros((B, n_q, H, d))
    for b in range(B):
        L = int(sl[b])
        for G in range(Hkv):
            for r in range(n_q):
                if flags & VISUAL_ONLY:
                    lo, hi = vb, vb + nv
                else:
                    lo, hi = 0, L - n_q + r + 1
                Kr = Kd[b, G, lo:hi]                       # [n][d]
                Vr = Vd[b, G, lo:hi]
                qr = qd[b, r, G * g:(G + 1) * g]            # [g][d]
                s = scale * (Kr @ qr.T)                     # [n][g]
                if li is None:
                    m = s.max(axis=0)
                    lr = m + np.log(np.exp(s - m).sum(axis=0))
                else:
                    lr = li[b, r, G * g:(G + 1) * g]
                p = np.exp(s - lr)                          # [n][g]
                out[b, r, G * g:(G + 1) * g] = p.T @ Vr
                absmass[b, r, G * g:(G + 1) * g] = p.T @ np.abs(Vr)
                lse[b, r, G * g:(G + 1) * g] = lr
    return out, lse, absmass


def pages_to_rows(page_idx, page: int):
    """Ascending page indices -> the ascending visual rows they cover (relative to vb)."""
    pi = np.asarray(page_idx, dtype=np.int64)
    rows = pi[..., :, None] * page + np.arange(page)[None, :]
    return rows.reshape(*pi.shape[:-1], pi.shape[-1] * page).astype(np.int32)


def mrope_plan(coords, vb: int, kept):
    """mRoPE remap plan (reading A23).  coords int [B][nv][3] (t, h, w);
    kept int [B][k] ascending.  Returns (new_coords int32 [B][k][3], text_start int32 [B])."""
    c = np.ascontiguousarray(np.asarray(coords, dtype=np.int32))
    kp = np.ascontiguousarray(np.asarray(kept, dtype=np.int32))
    B, nv, _ = c.shape
    k = kp.shape[-1]
    nc = np.zeros((B, k, 3), np.int32)
    ts = np.zeros((B,), np.int32)
    rc = lib().o_mrope_plan(_ptr(c), B, nv, vb, _ptr(kp), k, _ptr(nc), _ptr(ts))
    _check(rc, "o_mrope_plan")
    return nc, ts


def mrope_remap(K_pre, seq_len, vb: int, nv: int, kept, new_coords, text_start, sections, base: float,
                cap_out: int | None = None):
    """Apply the mRoPE plan (reading A23).  Returns (K_post float64 [B][Hkv][cap_out][d], rows)."""
    Kc = K_pre.contiguous()
    B, Hkv, cap, d = Kc.shape
    kp = np.ascontiguousarray(np.asarray(kept, dtype=np.int32))
    k = kp.shape[-1]
    sl = np.ascontiguousarray(np.asarray(seq_len, dtype=np.int32))
    nc = np.ascontiguousarray(np.asarray(new_coords, dtype=np.int32))
    ts = np.ascontiguousarray(np.asarray(text_start, dtype=np.int32))
    sec = np.ascontiguousarray(np.asarray(sections, dtype=np.int32))
    cap_out = cap - nv + k if cap_out is None else cap_out
    out = np.zeros((B, Hkv, cap_out, d), np.float64)
    rows = np.zeros((B, cap_out), np.int32)
    rc = lib().o_mrope_remap(_ptr(_u16(Kc)), B, Hkv, d, cap, _ptr(sl), vb, nv, _ptr(kp), k, _ptr(nc), _ptr(ts),
                             _ptr(sec), base, _ptr(out), cap_out, _ptr(rows))
    _check(rc, "o_mrope_remap")
    return out, rows
