"""Thin ctypes binding of libsparsevila.so (include/sparsevila.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  Tensors are torch CUDA tensors (PyTorch provides
device memory and streams).  There is no CPU fallback: if the library is
missing or a tensor is not on a CUDA device, the call raises.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SVL_LIB") or os.path.join(HERE, "libsparsevila.so")  # SVL_LIB: experiment builds

SVL_OK = 0
SVL_NORM_VISUAL_ONLY = 1
SVL_SELECT_SHARED = 2
SVL_RETRIEVE_SCORE_ONLY = 0x100
SVL_RETRIEVE_SELECT_ONLY = 0x200
SVL_FRESH_UNFUSED = 0x400
WORKSPACE_HEADER_BYTES = 1024  # SVL_WORKSPACE_HEADER_BYTES
SVL_IDX_PADDED = 0x800
SVL_SHARD_VIEW = 0x1000
SVL_DECODE_GRID_MERGE = 0x2000
SVL_DECODE_STATIC_PREFIX = 0x4000
SVL_PIN_SPLITS_MASK = 0xff000000


def SVL_PIN_SPLITS(n: int) -> int:
    """flags bits 24..31: pin the per-unit split count (include/sparsevila.h)."""
    return (int(n) & 0xff) << 24
SVL_SAL_SUMMARY, SVL_SAL_MULTI_SUMMARY, SVL_SAL_INTRA_VISUAL = 0, 1, 2
SVL_DEVFLAG_INDEX, SVL_DEVFLAG_NONFINITE, SVL_DEVFLAG_SPAN, SVL_DEVFLAG_WAIT_TIMEOUT = 1, 2, 4, 8

STATUS = {0: "SVL_OK", 1: "SVL_ERR_INVALID_ARGUMENT", 2: "SVL_ERR_SHAPE", 3: "SVL_ERR_ALIGNMENT",
          4: "SVL_ERR_WORKSPACE", 5: "SVL_ERR_UNSUPPORTED", 6: "SVL_ERR_CUDA"}

EXPORTS = ["svl_retrieve", "svl_retrieve_workspace_size", "svl_sparse_decode_attn",
           "svl_sparse_decode_workspace_size", "svl_fresh_decode_step",
           "svl_fresh_decode_workspace_size", "svl_prefill_prune", "svl_prune_workspace_size",
           "svl_salience", "svl_salience_workspace_size", "svl_keep_budget", "svl_workspace_init",
           "svl_status_string", "svl_last_error_message", "svl_read_device_flags",
           "svl_reset_device_flags", "svl_version", "svl_sparse_decode_attn_push",
           "svl_wait_flags", "svl_pack_kv", "svl_rope_remap", "svl_fresh_decode_plan",
           "svl_page_summary", "svl_retrieve_pages", "svl_retrieve_pages_workspace_size",
           "svl_mrope_remap", "svl_mrope_remap_workspace_size", "svl_retrieve_partial_lse",
           "svl_lse_combine", "svl_topk", "svl_topk_workspace_size", "svl_shard_indices", "svl_merge_partials",
           "svl_question_attention", "svl_question_attention_workspace_size"]


class SvlError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class svl_kv(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("stride_b", ctypes.c_int64),
                ("stride_h", ctypes.c_int64), ("stride_t", ctypes.c_int64),
                ("capacity", ctypes.c_int32)]


class svl_span(ctypes.Structure):
    _fields_ = [("visual_begin", ctypes.c_int32), ("visual_len", ctypes.c_int32),
                ("seq_len", ctypes.c_void_p)]


_lib = None


def lib():
    """Load libsparsevila.so (fails loudly; no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2510_17777_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, F, D, U32, SZ = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                      ctypes.c_float, ctypes.c_double, ctypes.c_uint32,
                                      ctypes.c_size_t)
        L.svl_retrieve.restype = ctypes.c_int
        L.svl_retrieve.argtypes = [P, I32, I32, I32, I32, I32, svl_kv, svl_span, P, I32, F, U32,
                                   P, P, P, SZ, P]
        L.svl_retrieve_workspace_size.restype = SZ
        L.svl_retrieve_workspace_size.argtypes = [I32, I32, I32, I32, I32, I32, U32]
        L.svl_question_attention.restype = ctypes.c_int
        L.svl_question_attention.argtypes = [P, I32, I32, I32, I32, I32, svl_kv, svl_kv, svl_span, P, F, U32,
                                             P, P, P, SZ, P]
        L.svl_question_attention_workspace_size.restype = SZ
        L.svl_question_attention_workspace_size.argtypes = [I32, I32, I32, I32, I32, I32, U32]
        if hasattr(L, "svl_rope_remap"):
            L.svl_rope_remap.restype = ctypes.c_int
            L.svl_rope_remap.argtypes = [svl_kv, svl_kv, I32, I32, I32, svl_span, P, I32, D, svl_kv, svl_kv,
                                         P, SZ, P]
        if hasattr(L, "svl_pack_kv"):  # (older experiment builds predate it; the ABI test checks it)
            L.svl_pack_kv.restype = ctypes.c_int
            L.svl_pack_kv.argtypes = [svl_kv, svl_kv, I32, I32, I32, svl_span, P, I32, U32, svl_kv, svl_kv,
                                      P, SZ, P]
        L.svl_sparse_decode_attn.restype = ctypes.c_int
        L.svl_sparse_decode_attn.argtypes = [P, I32, I32, I32, I32, svl_kv, svl_kv, svl_span, P,
                                             I32, U32, F, P, P, P, SZ, P]
        L.svl_sparse_decode_workspace_size.restype = SZ
        L.svl_sparse_decode_workspace_size.argtypes = [I32, I32, I32, I32, I32, I32, I32, U32]
        L.svl_fresh_decode_step.restype = ctypes.c_int
        L.svl_fresh_decode_step.argtypes = [P, I32, I32, I32, I32, svl_kv, svl_kv, svl_span, I32,
                                            F, U32, P, P, P, P, SZ, P]
        L.svl_retrieve_partial_lse.restype = ctypes.c_int
        L.svl_retrieve_partial_lse.argtypes = [P, I32, I32, I32, I32, I32, svl_kv, svl_span, ctypes.c_float, U32, P,
                                               P, SZ, P]
        L.svl_lse_combine.restype = ctypes.c_int
        L.svl_lse_combine.argtypes = [P, I32, I32, P, P]
        L.svl_topk.restype = ctypes.c_int
        L.svl_topk.argtypes = [P, I32, I32, I32, P, P, SZ, P]
        L.svl_topk_workspace_size.restype = SZ
        L.svl_topk_workspace_size.argtypes = [I32, I32]
        L.svl_shard_indices.restype = ctypes.c_int
        L.svl_shard_indices.argtypes = [P, I32, I32, I32, I32, P, P]
        L.svl_merge_partials.restype = ctypes.c_int
        L.svl_merge_partials.argtypes = [P, P, I32, I32, I32, P, P, P]
        L.svl_mrope_remap.restype = ctypes.c_int
        L.svl_mrope_remap.argtypes = [svl_kv, svl_kv, I32, I32, I32, svl_span, P, P, I32, ctypes.c_double, P,
                                      svl_kv, svl_kv, P, P, P, SZ, P]
        L.svl_mrope_remap_workspace_size.restype = SZ
        L.svl_mrope_remap_workspace_size.argtypes = [I32, I32]
        L.svl_page_summary.restype = ctypes.c_int
        L.svl_page_summary.argtypes = [svl_kv, I32, I32, I32, svl_span, I32, P, P, P, SZ, P]
        L.svl_retrieve_pages.restype = ctypes.c_int
        L.svl_retrieve_pages.argtypes = [P, I32, I32, I32, I32, I32, P, P, I32, I32, I32, ctypes.c_float, U32,
                                         P, P, P, P, SZ, P]
        L.svl_retrieve_pages_workspace_size.restype = SZ
        L.svl_retrieve_pages_workspace_size.argtypes = [I32, I32, I32, I32, I32]
        L.svl_fresh_decode_plan.restype = ctypes.c_int
        L.svl_fresh_decode_plan.argtypes = [I32, I32, I32, I32, I32, I32, U32]
        L.svl_fresh_decode_workspace_size.restype = SZ
        L.svl_fresh_decode_workspace_size.argtypes = [I32, I32, I32, I32, I32, I32, I32, U32]
        L.svl_prefill_prune.restype = ctypes.c_int
        L.svl_prefill_prune.argtypes = [P, I32, I32, P, I32, D, P, I32, P, P, SZ, P]
        L.svl_prune_workspace_size.restype = SZ
        L.svl_prune_workspace_size.argtypes = [I32, I32, I32]
        L.svl_salience.restype = ctypes.c_int
        L.svl_salience.argtypes = [P, P, I32, I32, I32, I32, I32, I32, F, P, P, SZ, P]
        L.svl_salience_workspace_size.restype = SZ
        L.svl_salience_workspace_size.argtypes = [I32, I32, I32, I32, I32, I32]
        L.svl_keep_budget.restype = I64
        L.svl_keep_budget.argtypes = [I64, D]
        L.svl_workspace_init.restype = ctypes.c_int
        L.svl_workspace_init.argtypes = [P, SZ, P]
        L.svl_status_string.restype = ctypes.c_char_p
        L.svl_status_string.argtypes = [ctypes.c_int]
        L.svl_last_error_message.restype = ctypes.c_char_p
        L.svl_last_error_message.argtypes = []
        L.svl_read_device_flags.restype = ctypes.c_int
        L.svl_read_device_flags.argtypes = [P, P, P]
        L.svl_reset_device_flags.restype = ctypes.c_int
        L.svl_reset_device_flags.argtypes = [P, P]
        L.svl_version.restype = ctypes.c_char_p
        L.svl_version.argtypes = []
        L.svl_sparse_decode_attn_push.restype = ctypes.c_int
        L.svl_sparse_decode_attn_push.argtypes = [P, I32, I32, I32, I32, svl_kv, svl_kv, svl_span, P,
                                                  I32, U32, F, P, P, P, P, I32, I32, U32, I32, I32,
                                                  I32, I32, P, SZ, P]
        L.svl_wait_flags.restype = ctypes.c_int
        L.svl_wait_flags.argtypes = [P, I32, U32, P, P]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != SVL_OK:
        raise SvlError(rc, lib().svl_last_error_message().decode())


def _cuda(t: torch.Tensor, name: str, dtype=None) -> int:
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def kv_view(t: torch.Tensor, name: str = "K") -> svl_kv:
    """[B][Hkv][cap][d] bf16 CUDA tensor (last dim contiguous) -> svl_kv."""
    _cuda(t, name, torch.bfloat16)
    if t.dim() != 4 or t.stride(3) != 1:
        raise ValueError(f"{name} must be [B][Hkv][cap][d] with a contiguous last dim")
    return svl_kv(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2), t.shape[2])


def span(visual_begin: int, visual_len: int, seq_len: torch.Tensor) -> svl_span:
    _cuda(seq_len, "seq_len", torch.int32)
    return svl_span(visual_begin, visual_len, seq_len.data_ptr())


class Workspace:
    """A zero-initialised device workspace (grown on demand)."""

    def __init__(self, device=None):
        self.buf: Optional[torch.Tensor] = None
        self.device = device

    def get(self, nbytes: int, stream=None) -> torch.Tensor:
        nbytes = max(int(nbytes), WORKSPACE_HEADER_BYTES)
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=self.device or "cuda")
        return self.buf

    def flags(self, stream=None) -> int:
        if self.buf is None:  # never used: nothing raised
            return 0
        out = ctypes.c_uint32(0)
        _check(lib().svl_read_device_flags(ctypes.c_void_p(self.buf.data_ptr()),
                                           ctypes.c_void_p(_stream(stream)), ctypes.byref(out)))
        return out.value

    def reset_flags(self, stream=None):
        if self.buf is None:
            return
        _check(lib().svl_reset_device_flags(ctypes.c_void_p(self.buf.data_ptr()),
                                            ctypes.c_void_p(_stream(stream))))


_default_ws = {}


def _ws(ws: Optional[Workspace], device) -> Workspace:
    if ws is not None:
        return ws
    key = str(device)
    if key not in _default_ws:
        _default_ws[key] = Workspace(device)
    return _default_ws[key]


def keep_budget(n: int, s: float) -> int:
    return int(lib().svl_keep_budget(n, s))


def retrieve_workspace_size(B, n_q, H, Hkv, d, visual_len, flags=0) -> int:
    return int(lib().svl_retrieve_workspace_size(B, n_q, H, Hkv, d, visual_len, flags))


def sparse_decode_workspace_size(B, H, Hkv, d, k, visual_len, capacity, flags=0) -> int:
    return int(lib().svl_sparse_decode_workspace_size(B, H, Hkv, d, k, visual_len, capacity, flags))


def retrieve(q: torch.Tensor, K: torch.Tensor, seq_len: torch.Tensor, visual_begin: int,
             visual_len: int, k: int, scale: Optional[float] = None, flags: int = 0,
             lse_in: Optional[torch.Tensor] = None, idx_out: Optional[torch.Tensor] = None,
             scores_out: Optional[torch.Tensor] = None, ws: Optional[Workspace] = None,
             stream=None) -> torch.Tensor:
    """svl_retrieve.  q bf16 [B][n_q][H][d]; K bf16 [B][Hkv][cap][d]; returns
    int32 [B][U][k] ascending visual indices (U = Hkv, or 1 with SHARED)."""
    B, n_q, H, d = q.shape
    Hkv = K.shape[1]
    U = 1 if flags & SVL_SELECT_SHARED else Hkv
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    _cuda(q, "q", torch.bfloat16)
    if not q.is_contiguous():
        raise ValueError("q must be contiguous")
    if idx_out is None:
        idx_out = torch.empty(B, U, max(k, 0), dtype=torch.int32, device=q.device)
    wsz = retrieve_workspace_size(B, n_q, H, Hkv, d, visual_len, flags)
    w = _ws(ws, q.device).get(wsz)
    _check(lib().svl_retrieve(
        q.data_ptr(), B, n_q, H, Hkv, d, kv_view(K), span(visual_begin, visual_len, seq_len),
        _cuda(lse_in, "lse_in", torch.float32) if lse_in is not None else None, k, scale, flags,
        _cuda(idx_out, "idx_out", torch.int32),
        _cuda(scores_out, "scores_out", torch.float32) if scores_out is not None else None,
        w.data_ptr(), w.numel(), _stream(stream)))
    return idx_out


def question_attention_workspace_size(B, n_q, H, Hkv, d, visual_len, flags=0) -> int:
    return int(lib().svl_question_attention_workspace_size(B, n_q, H, Hkv, d, visual_len, flags))


def question_attention(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, seq_len: torch.Tensor,
                       visual_begin: int, visual_len: int, scale: Optional[float] = None, flags: int = 0,
                       lse_in: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                       lse_out: Optional[torch.Tensor] = None, ws: Optional[Workspace] = None, stream=None):
    """svl_question_attention (the question chunk's attention output).
    q bf16 [B][n_q][H][d]; K, V bf16 [B][Hkv][cap][d].  Returns (out fp32 [B][n_q][H][d],
    lse fp32 [B][n_q][H] natural log)."""
    B, n_q, H, d = q.shape
    Hkv = K.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    _cuda(q, "q", torch.bfloat16)
    if not q.is_contiguous():
        raise ValueError("q must be contiguous")
    if out is None:
        out = torch.empty(B, n_q, H, d, dtype=torch.float32, device=q.device)
    if lse_out is None:
        lse_out = torch.empty(B, n_q, H, dtype=torch.float32, device=q.device)
    w = _ws(ws, q.device).get(question_attention_workspace_size(B, n_q, H, Hkv, d, visual_len, flags))
    _check(lib().svl_question_attention(
        q.data_ptr(), B, n_q, H, Hkv, d, kv_view(K), kv_view(V, "V"), span(visual_begin, visual_len, seq_len),
        _cuda(lse_in, "lse_in", torch.float32) if lse_in is not None else None, scale, flags,
        _cuda(out, "out", torch.float32), _cuda(lse_out, "lse_out", torch.float32),
        w.data_ptr(), w.numel(), _stream(stream)))
    return out, lse_out


def rope_remap(K_pre: torch.Tensor, V: Optional[torch.Tensor], seq_len: torch.Tensor, visual_begin: int,
               visual_len: int, kept: torch.Tensor, rope_base: float = 10000.0,
               K_out: Optional[torch.Tensor] = None, V_out: Optional[torch.Tensor] = None,
               ws: Optional[Workspace] = None, stream=None):
    """svl_rope_remap (unified RoPE remap after pruning).
    kept int32 [B][k] relative to visual_begin.  Returns (K_out, V_out or None, seq_len_new)."""
    B, Hkv, cap, d = K_pre.shape
    k = kept.shape[-1]
    ocap = visual_begin + k + (cap - visual_begin - visual_len)
    if K_out is None:
        K_out = torch.zeros(B, Hkv, ocap, d, dtype=K_pre.dtype, device=K_pre.device)
    if V is not None and V_out is None:
        V_out = torch.zeros(B, Hkv, ocap, d, dtype=V.dtype, device=V.device)
    null_kv = svl_kv(None, 0, 0, 0, 0)
    w = _ws(ws, K_pre.device).get(WORKSPACE_HEADER_BYTES)
    _check(lib().svl_rope_remap(kv_view(K_pre, "K_pre"), kv_view(V, "V") if V is not None else null_kv, B, Hkv, d,
                                span(visual_begin, visual_len, seq_len), _cuda(kept, "kept", torch.int32), k,
                                float(rope_base), kv_view(K_out, "K_out"),
                                kv_view(V_out, "V_out") if V is not None else null_kv,
                                w.data_ptr(), w.numel(), _stream(stream)))
    return K_out, V_out, (seq_len - visual_len + k).to(torch.int32)


def pack_kv(K: torch.Tensor, V: torch.Tensor, seq_len: torch.Tensor, visual_begin: int,
            visual_len: int, vis_idx: torch.Tensor, flags: int = 0, Kp: Optional[torch.Tensor] = None,
            Vp: Optional[torch.Tensor] = None, ws: Optional[Workspace] = None, stream=None):
    """svl_pack_kv (pack-once).  Returns (Kp, Vp, seq_len_packed):
    the packed caches [B][Hkv][vb + k + cap - vb - N_v][d] and seq_len - N_v + k."""
    B, Hkv, cap, d = K.shape
    k = vis_idx.shape[-1]
    pcap = visual_begin + k + (cap - visual_begin - visual_len)
    if Kp is None:
        Kp = torch.empty(B, Hkv, pcap, d, dtype=K.dtype, device=K.device)
    if Vp is None:
        Vp = torch.empty(B, Hkv, pcap, d, dtype=V.dtype, device=V.device)
    w = _ws(ws, K.device).get(WORKSPACE_HEADER_BYTES)
    _check(lib().svl_pack_kv(kv_view(K, "K"), kv_view(V, "V"), B, Hkv, d,
                             span(visual_begin, visual_len, seq_len),
                             _cuda(vis_idx, "vis_idx", torch.int32), k, flags, kv_view(Kp, "Kp"),
                             kv_view(Vp, "Vp"), w.data_ptr(), w.numel(), _stream(stream)))
    return Kp, Vp, (seq_len - visual_len + k).to(torch.int32)


def sparse_decode_attn(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, seq_len: torch.Tensor,
                       visual_begin: int, visual_len: int, vis_idx: Optional[torch.Tensor],
                       scale: Optional[float] = None, flags: int = 0,
                       out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None,
                       ws: Optional[Workspace] = None, stream=None):
    """svl_sparse_decode_attn.  q bf16 [B][H][d]; vis_idx int32 [B][U][k].
    Returns (out fp32 [B][H][d], lse fp32 [B][H] or None)."""
    B, H, d = q.shape
    Hkv = K.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    _cuda(q, "q", torch.bfloat16)
    if not q.is_contiguous():
        raise ValueError("q must be contiguous")
    k = 0 if vis_idx is None else vis_idx.shape[-1]
    if out is None:
        out = torch.empty(B, H, d, dtype=torch.float32, device=q.device)
    wsz = sparse_decode_workspace_size(B, H, Hkv, d, k, visual_len, K.shape[2], flags)
    w = _ws(ws, q.device).get(wsz)
    _check(lib().svl_sparse_decode_attn(
        q.data_ptr(), B, H, Hkv, d, kv_view(K, "K"), kv_view(V, "V"),
        span(visual_begin, visual_len, seq_len),
        _cuda(vis_idx, "vis_idx", torch.int32) if vis_idx is not None else None, k, flags, scale,
        _cuda(out, "out", torch.float32),
        _cuda(lse_out, "lse_out", torch.float32) if lse_out is not None else None,
        w.data_ptr(), w.numel(), _stream(stream)))
    return out, lse_out


def sparse_decode_attn_push(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, seq_len: torch.Tensor,
                            visual_begin: int, visual_len: int, vis_idx: Optional[torch.Tensor],
                            peer_out, peer_flags, rank: int, epoch: int, b0: int, h0: int,
                            scale: Optional[float] = None, flags: int = 0,
                            out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None,
                            ws: Optional[Workspace] = None, stream=None):
    """svl_sparse_decode_attn_push: this rank's shard of the decode, stored into every
    rank's gathered output peer_out[r] (fp32 [B_total][H_total][d]) and flagged in
    peer_flags[r] (uint32 [P]) with `epoch`.  Returns out (local copy or None)."""
    B, H, d = q.shape
    Hkv = K.shape[1]
    P = len(peer_out)
    if len(peer_flags) != P:
        raise ValueError("peer_out and peer_flags must have one entry per rank")
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    _cuda(q, "q", torch.bfloat16)
    if not q.is_contiguous():
        raise ValueError("q must be contiguous")
    k = 0 if vis_idx is None else vis_idx.shape[-1]
    B_total, H_total = peer_out[0].shape[0], peer_out[0].shape[1]
    po = (ctypes.c_void_p * P)(*[_cuda(t, "peer_out", torch.float32) for t in peer_out])
    pf = (ctypes.c_void_p * P)(*[_cuda(t, "peer_flags", torch.int32) for t in peer_flags])
    wsz = sparse_decode_workspace_size(B, H, Hkv, d, k, visual_len, K.shape[2], flags)
    w = _ws(ws, q.device).get(wsz)
    _check(lib().svl_sparse_decode_attn_push(
        q.data_ptr(), B, H, Hkv, d, kv_view(K, "K"), kv_view(V, "V"),
        span(visual_begin, visual_len, seq_len),
        _cuda(vis_idx, "vis_idx", torch.int32) if vis_idx is not None else None, k, flags, scale,
        _cuda(out, "out", torch.float32) if out is not None else None,
        _cuda(lse_out, "lse_out", torch.float32) if lse_out is not None else None,
        ctypes.cast(po, ctypes.c_void_p), ctypes.cast(pf, ctypes.c_void_p), rank, P, epoch, b0, h0,
        B_total, H_total, w.data_ptr(), w.numel(), _stream(stream)))
    return out


def wait_flags(flags: torch.Tensor, epoch: int, ws: Optional[Workspace] = None, stream=None):
    """svl_wait_flags: stream-ordered wait until flags[s] >= epoch for all s (int32 [P] tensor)."""
    w = _ws(ws, flags.device).get(WORKSPACE_HEADER_BYTES)
    _check(lib().svl_wait_flags(_cuda(flags, "flags", torch.int32), flags.numel(), epoch,
                                w.data_ptr(), _stream(stream)))


def fresh_uses_fused(B, H, Hkv, d, visual_len, capacity, flags=0) -> bool:
    """Whether svl_fresh_decode_step runs the fused kernel (one launch per call) for a shape."""
    return bool(lib().svl_fresh_decode_plan(B, H, Hkv, d, visual_len, capacity, flags))


def fresh_decode_workspace_size(B, H, Hkv, d, k, visual_len, capacity, flags=0) -> int:
    return int(lib().svl_fresh_decode_workspace_size(B, H, Hkv, d, k, visual_len, capacity, flags))


def fresh_decode_step(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, seq_len: torch.Tensor,
                      visual_begin: int, visual_len: int, k: int, scale: Optional[float] = None,
                      flags: int = 0, idx_out: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None, lse_out: Optional[torch.Tensor] = None,
                      ws: Optional[Workspace] = None, stream=None):
    """svl_fresh_decode_step (fused retrieve + sparse decode, same query).
    q bf16 [B][H][d].  Returns (out fp32 [B][H][d], idx int32 [B][Hkv][k])."""
    B, H, d = q.shape
    Hkv = K.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    _cuda(q, "q", torch.bfloat16)
    if not q.is_contiguous():
        raise ValueError("q must be contiguous")
    if idx_out is None:
        idx_out = torch.empty(B, Hkv, max(k, 0), dtype=torch.int32, device=q.device)
    if out is None:
        out = torch.empty(B, H, d, dtype=torch.float32, device=q.device)
    wsz = fresh_decode_workspace_size(B, H, Hkv, d, k, visual_len, K.shape[2], flags)
    w = _ws(ws, q.device).get(wsz)
    _check(lib().svl_fresh_decode_step(
        q.data_ptr(), B, H, Hkv, d, kv_view(K, "K"), kv_view(V, "V"),
        span(visual_begin, visual_len, seq_len), k, scale, flags,
        _cuda(idx_out, "idx_out", torch.int32), _cuda(out, "out", torch.float32),
        _cuda(lse_out, "lse_out", torch.float32) if lse_out is not None else None,
        w.data_ptr(), w.numel(), _stream(stream)))
    return out, idx_out


def prefill_prune(saliency: torch.Tensor, prefill_sparsity: float, frame_offsets=None,
                  kept_idx: Optional[torch.Tensor] = None, ws: Optional[Workspace] = None,
                  stream=None):
    """svl_prefill_prune.  saliency fp32 [B][N] (CUDA); frame_offsets: host
    sequence of n_frames+1 ints or None.  Returns (kept int32 [B][total], total)."""
    _cuda(saliency, "saliency", torch.float32)
    B, N = saliency.shape
    if frame_offsets is not None:
        fo = (ctypes.c_int32 * len(frame_offsets))(*[int(x) for x in frame_offsets])
        nf = len(frame_offsets) - 1
        cap = sum(max(keep_budget(int(frame_offsets[i + 1]) - int(frame_offsets[i]),
                                  prefill_sparsity), 0) for i in range(nf))
    else:
        fo, nf = None, 1
        cap = keep_budget(N, prefill_sparsity)
    cap = max(cap, 1)
    if kept_idx is None:
        kept_idx = torch.empty(B, cap, dtype=torch.int32, device=saliency.device)
    total = ctypes.c_int32(0)
    w = _ws(ws, saliency.device).get(lib().svl_prune_workspace_size(B, N, nf))
    _check(lib().svl_prefill_prune(
        saliency.data_ptr(), B, N, ctypes.cast(fo, ctypes.c_void_p) if fo is not None else None,
        nf, float(prefill_sparsity), _cuda(kept_idx, "kept_idx", torch.int32), kept_idx.shape[1],
        ctypes.addressof(total), w.data_ptr(), w.numel(), _stream(stream)))
    return kept_idx[:, :total.value], total.value


def salience(Qe: torch.Tensor, Ke: torch.Tensor, S: int, mode: int,
             scale: Optional[float] = None, out: Optional[torch.Tensor] = None,
             ws: Optional[Workspace] = None, stream=None) -> torch.Tensor:
    """svl_salience.  Qe, Ke bf16 [F][S+N_f][H_e][d_e] -> fp32 [F][N_f]."""
    _cuda(Qe, "Qe", torch.bfloat16)
    _cuda(Ke, "Ke", torch.bfloat16)
    if not (Qe.is_contiguous() and Ke.is_contiguous()):
        raise ValueError("Qe, Ke must be contiguous")
    F, T, He, de = Qe.shape
    Nf = T - S
    if scale is None:
        scale = 1.0 / math.sqrt(de)
    if out is None:
        out = torch.empty(F, Nf, dtype=torch.float32, device=Qe.device)
    w = _ws(ws, Qe.device).get(lib().svl_salience_workspace_size(F, S, Nf, He, de, mode))
    _check(lib().svl_salience(Qe.data_ptr(), Ke.data_ptr(), F, S, Nf, He, de, mode, scale,
                              _cuda(out, "out", torch.float32), w.data_ptr(), w.numel(),
                              _stream(stream)))
    return out


def version() -> str:
    return lib().svl_version().decode()


def page_summary(K: torch.Tensor, visual_begin: int, visual_len: int, page: int,
                 kmax: Optional[torch.Tensor] = None, kmin: Optional[torch.Tensor] = None,
                 ws: Optional[Workspace] = None, stream=None):
    """svl_page_summary.  K bf16 [B][Hkv][cap][d] -> (kmax, kmin) bf16 [B][Hkv][visual_len/page][d]."""
    B, Hkv, _, d = K.shape
    npg = visual_len // page
    if kmax is None:
        kmax = torch.empty(B, Hkv, npg, d, dtype=torch.bfloat16, device=K.device)
    if kmin is None:
        kmin = torch.empty(B, Hkv, npg, d, dtype=torch.bfloat16, device=K.device)
    w = _ws(ws, K.device).get(WORKSPACE_HEADER_BYTES)
    seq = torch.full((B,), visual_begin + visual_len, dtype=torch.int32, device=K.device)
    _check(lib().svl_page_summary(kv_view(K, "K"), B, Hkv, d, span(visual_begin, visual_len, seq), page,
                                  _cuda(kmax, "kmax", torch.bfloat16), _cuda(kmin, "kmin", torch.bfloat16),
                                  w.data_ptr(), w.numel(), _stream(stream)))
    return kmax, kmin


def retrieve_pages(q: torch.Tensor, kmax: torch.Tensor, kmin: torch.Tensor, page: int, k_pages: int,
                   scale: Optional[float] = None, page_idx_out: Optional[torch.Tensor] = None,
                   row_idx_out: Optional[torch.Tensor] = None, scores_out: Optional[torch.Tensor] = None,
                   want_rows: bool = True, ws: Optional[Workspace] = None, stream=None):
    """svl_retrieve_pages.  q bf16 [B][n_q][H][d].  Returns (page_idx [B][Hkv][k_pages],
    rows [B][Hkv][k_pages * page] or None)."""
    B, n_q, H, d = q.shape
    _, Hkv, npg, _ = kmax.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    _cuda(q, "q", torch.bfloat16)
    if not (q.is_contiguous() and kmax.is_contiguous() and kmin.is_contiguous()):
        raise ValueError("q, kmax, kmin must be contiguous")
    if page_idx_out is None:
        page_idx_out = torch.empty(B, Hkv, k_pages, dtype=torch.int32, device=q.device)
    if row_idx_out is None and want_rows:
        row_idx_out = torch.empty(B, Hkv, k_pages * page, dtype=torch.int32, device=q.device)
    w = _ws(ws, q.device).get(lib().svl_retrieve_pages_workspace_size(B, n_q, H, Hkv, npg))
    _check(lib().svl_retrieve_pages(
        q.data_ptr(), B, n_q, H, Hkv, d, _cuda(kmax, "kmax", torch.bfloat16), _cuda(kmin, "kmin", torch.bfloat16),
        npg, page, k_pages, scale, 0, _cuda(page_idx_out, "page_idx_out", torch.int32),
        _cuda(row_idx_out, "row_idx_out", torch.int32) if row_idx_out is not None else None,
        _cuda(scores_out, "scores_out", torch.float32) if scores_out is not None else None,
        w.data_ptr(), w.numel(), _stream(stream)))
    return page_idx_out, row_idx_out


def mrope_remap(K_pre: torch.Tensor, V: Optional[torch.Tensor], seq_len: torch.Tensor, visual_begin: int,
                visual_len: int, coords: torch.Tensor, kept: torch.Tensor, rope_base: float, sections,
                K_out: Optional[torch.Tensor] = None, V_out: Optional[torch.Tensor] = None,
                ws: Optional[Workspace] = None, stream=None):
    """svl_mrope_remap.  coords int32 [B][visual_len][3]; kept int32 [B][k]; sections 3 ints.
    Returns (K_out, V_out, new_coords int32 [B][k][3], text_start int32 [B])."""
    B, Hkv, cap, d = K_pre.shape
    k = kept.shape[-1]
    cap_out = cap - visual_len + k
    if K_out is None:
        K_out = torch.empty(B, Hkv, cap_out, d, dtype=torch.bfloat16, device=K_pre.device)
    if V is not None and V_out is None:
        V_out = torch.empty(B, Hkv, cap_out, d, dtype=torch.bfloat16, device=K_pre.device)
    nc = torch.empty(B, k, 3, dtype=torch.int32, device=K_pre.device)
    ts = torch.empty(B, dtype=torch.int32, device=K_pre.device)
    sec = (ctypes.c_int32 * 3)(*[int(x) for x in sections])
    w = _ws(ws, K_pre.device).get(lib().svl_mrope_remap_workspace_size(B, k))
    empty = svl_kv(None, 0, 0, 0, 0)
    _check(lib().svl_mrope_remap(
        kv_view(K_pre, "K_pre"), kv_view(V, "V") if V is not None else empty, B, Hkv, d,
        span(visual_begin, visual_len, seq_len), _cuda(coords.contiguous(), "coords", torch.int32),
        _cuda(kept.contiguous(), "kept", torch.int32), k, float(rope_base), ctypes.cast(sec, ctypes.c_void_p),
        kv_view(K_out, "K_out"), kv_view(V_out, "V_out") if V_out is not None else empty,
        nc.data_ptr(), ts.data_ptr(), w.data_ptr(), w.numel(), _stream(stream)))
    return K_out, V_out, nc, ts


# ------------------------------------------- sequence split

def retrieve_partial_lse(q: torch.Tensor, K: torch.Tensor, seq_len: torch.Tensor, visual_begin: int,
                         visual_len: int, flags: int = 0, scale: Optional[float] = None,
                         lse_out: Optional[torch.Tensor] = None, ws: Optional[Workspace] = None, stream=None):
    """svl_retrieve_partial_lse.  q bf16 [B][n_q][H][d] -> natural-log LSE fp32 [B][n_q][H]."""
    B, n_q, H, d = q.shape
    Hkv = K.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    _cuda(q, "q", torch.bfloat16)
    if lse_out is None:
        lse_out = torch.empty(B, n_q, H, dtype=torch.float32, device=q.device)
    w = _ws(ws, q.device).get(retrieve_workspace_size(B, n_q, H, Hkv, d, visual_len, flags & SVL_NORM_VISUAL_ONLY))
    _check(lib().svl_retrieve_partial_lse(q.data_ptr(), B, n_q, H, Hkv, d, kv_view(K, "K"),
                                          span(visual_begin, visual_len, seq_len), scale, flags,
                                          _cuda(lse_out, "lse_out", torch.float32), w.data_ptr(), w.numel(),
                                          _stream(stream)))
    return lse_out


def lse_combine(parts: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """svl_lse_combine.  parts fp32 [P][...] -> [...] (log-sum-exp over P in rank order)."""
    parts = parts.contiguous()
    P = parts.shape[0]
    if out is None:
        out = torch.empty(parts.shape[1:], dtype=torch.float32, device=parts.device)
    _check(lib().svl_lse_combine(_cuda(parts, "parts", torch.float32), P, parts[0].numel(),
                                 _cuda(out, "out", torch.float32), _stream(stream)))
    return out


def topk(scores: torch.Tensor, k: int, idx_out: Optional[torch.Tensor] = None, ws: Optional[Workspace] = None,
         stream=None) -> torch.Tensor:
    """svl_topk.  scores fp32 [units][n] -> ascending indices int32 [units][k] (ties -> lower index)."""
    scores = scores.contiguous()
    units, n = scores.shape
    if idx_out is None:
        idx_out = torch.empty(units, k, dtype=torch.int32, device=scores.device)
    w = _ws(ws, scores.device).get(lib().svl_topk_workspace_size(units, n))
    _check(lib().svl_topk(_cuda(scores, "scores", torch.float32), units, n, k, _cuda(idx_out, "idx_out", torch.int32),
                          w.data_ptr(), w.numel(), _stream(stream)))
    return idx_out


def shard_indices(idx: torch.Tensor, lo: int, hi: int, out: Optional[torch.Tensor] = None, stream=None):
    """svl_shard_indices.  idx int32 [..., k] ascending -> this shard's entries minus lo, -1 padded."""
    idx = idx.contiguous()
    k = idx.shape[-1]
    units = idx.numel() // max(k, 1)
    if out is None:
        out = torch.empty_like(idx)
    _check(lib().svl_shard_indices(_cuda(idx, "idx", torch.int32), units, k, lo, hi, _cuda(out, "out", torch.int32),
                                   _stream(stream)))
    return out


def merge_partials(out_parts: torch.Tensor, lse_parts: torch.Tensor, out: Optional[torch.Tensor] = None,
                   lse_out: Optional[torch.Tensor] = None, stream=None):
    """svl_merge_partials.  out_parts fp32 [P][...][d], lse_parts fp32 [P][...] -> (out, lse)."""
    out_parts = out_parts.contiguous()
    lse_parts = lse_parts.contiguous()
    P, d = out_parts.shape[0], out_parts.shape[-1]
    rows = lse_parts[0].numel()
    if out is None:
        out = torch.empty(out_parts.shape[1:], dtype=torch.float32, device=out_parts.device)
    if lse_out is None:
        lse_out = torch.empty(lse_parts.shape[1:], dtype=torch.float32, device=out_parts.device)
    _check(lib().svl_merge_partials(_cuda(out_parts, "out_parts", torch.float32),
                                    _cuda(lse_parts, "lse_parts", torch.float32), P, rows, d,
                                    _cuda(out, "out", torch.float32), _cuda(lse_out, "lse_out", torch.float32),
                                    _stream(stream)))
    return out, lse_out
