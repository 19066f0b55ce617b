"""CPU-side tests (-m "not gpu"): the C-ABI library loads and exports every
symbol include/sparsevila.h declares; host-side validation rejects bad
arguments before touching the device; the parity checker rejects corrupted
results (SURVEY.md 8(c) c6 "checker self-test")."""
import ctypes
import os
import re

import numpy as np
import pytest

from tests import parity

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def svl():
    from paper_2510_17777_b200 import build, svl as mod
    build.build()
    mod.lib()
    return mod


def _declared():
    src = open(os.path.join(ROOT, "include", "sparsevila.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(svl_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(svl):
    names = _declared()
    assert len(names) >= 14
    L = svl.lib()
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(svl.EXPORTS)


def test_library_is_sm100a_only(svl):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {svl.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out and "sm_90" not in out


def test_keep_budget_abi_matches_spec(svl):
    import json
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))
    for n, s, k in gold["P4_keep_budget"]["cases"]:
        assert svl.keep_budget(n, s) == k
    assert svl.keep_budget(5, 1.0) == -1 and svl.keep_budget(-1, 0.5) == -1


def test_status_strings(svl):
    L = svl.lib()
    for code, name in svl.STATUS.items():
        assert L.svl_status_string(code).decode() == name


def test_workspace_sizes_are_linear_not_quadratic(svl):
    L = svl.lib()
    a = L.svl_salience_workspace_size(1, 0, 1024, 16, 72, 2)
    b = L.svl_salience_workspace_size(1, 0, 4096, 16, 72, 2)
    assert 0 < a < b <= 4 * a + 4096          # O(N), never O(N^2)
    r = L.svl_retrieve_workspace_size(1, 1, 28, 4, 128, 32768, 0)
    assert 0 < r < 16 << 20
    assert L.svl_sparse_decode_workspace_size(1, 28, 4, 128, 3277, 32768, 33584, 0) > 0


def _kv(cap=100, d=128):
    return svl_mod().svl_kv(0x1000, 4 * cap * d, cap * d, d, cap)


def svl_mod():
    from paper_2510_17777_b200 import svl
    return svl


@pytest.mark.parametrize("case,status", [
    ("k_gt_nv", 1), ("h_mod", 2), ("no_visual", 2), ("bad_d", 5), ("misaligned_q", 3),
    ("null_ws", 4), ("bad_flags", 1), ("span_capacity", 2), ("big_group", 5)])
def test_retrieve_host_validation(svl, case, status):
    L = svl.lib()
    P = 0x10000
    args = dict(q=P, B=1, n_q=1, H=28, Hkv=4, d=128, K=_kv(), sp=svl.svl_span(10, 60, P), lse=None,
                k=10, scale=0.088, flags=0, idx=P, sc=None, ws=P, wsb=1 << 30, st=None)
    if case == "k_gt_nv":
        args["k"] = 61
    elif case == "h_mod":
        args["H"] = 27
    elif case == "no_visual":
        args["sp"] = svl.svl_span(10, 0, P)
    elif case == "bad_d":
        args["d"] = 96
        args["K"] = _kv(d=96)
    elif case == "misaligned_q":
        args["q"] = P + 2
    elif case == "null_ws":
        args["ws"] = None
    elif case == "bad_flags":
        args["flags"] = 8
    elif case == "span_capacity":
        args["sp"] = svl.svl_span(50, 60, P)
    elif case == "big_group":
        args["n_q"] = 600           # n_q * g = 4200 > 4096 query rows per unit
        args["K"] = _kv(cap=1000)
    rc = L.svl_retrieve(*args.values())
    assert rc == status, (rc, L.svl_last_error_message())
    assert L.svl_last_error_message()


def test_prune_host_validation(svl):
    L = svl.lib()
    P = 0x10000
    tot = ctypes.c_int32(-1)
    fo = (ctypes.c_int32 * 3)(0, 5, 9)            # does not end at N = 10
    rc = L.svl_prefill_prune(P, 1, 10, ctypes.cast(fo, ctypes.c_void_p), 2, 0.5, P, 100,
                             ctypes.addressof(tot), P, 1 << 20, None)
    assert rc == 2
    rc = L.svl_prefill_prune(P, 1, 10, None, 1, 1.0, P, 100, ctypes.addressof(tot), P, 1 << 20, None)
    assert rc == 1
    rc = L.svl_prefill_prune(P, 1, 10, None, 1, 0.5, P, 4, ctypes.addressof(tot), P, 1 << 20, None)
    assert rc == 1 and tot.value == -1             # capacity 4 < keep_budget(10, .5) = 5


def test_salience_mode_mismatch_rejected(svl):
    L = svl.lib()
    P = 0x10000
    assert L.svl_salience(P, P, 1, 1, 16, 2, 64, 2, 0.125, P, P, 1 << 20, None) == 1
    assert L.svl_salience(P, P, 1, 0, 16, 2, 64, 0, 0.125, P, P, 1 << 20, None) == 1
    assert L.svl_salience(P, P, 1, 0, 16, 2, 60, 2, 0.125, P, P, 1 << 20, None) == 5


# ------------------------------------------------------------ checker self-test


def _case():
    rng = np.random.default_rng(0)
    s = rng.random((1, 1, 200))
    k = 20
    order = np.lexsort((np.arange(200), -s[0, 0]))
    idx = np.sort(order[:k])[None, None]
    gap = np.array([[(s[0, 0, order[k - 1]] - s[0, 0, order[k]]) / s[0, 0, order[k - 1]]]])
    return s, idx, gap, k, order


def test_checker_accepts_the_truth():
    s, idx, gap, k, _ = _case()
    assert parity.check_indices(idx, s, gap, k) in (0.0, 1.0)


def test_checker_rejects_swapped_index():
    s, idx, gap, k, order = _case()
    bad = idx.copy()
    bad[0, 0, 0] = order[150]
    bad[0, 0] = np.sort(bad[0, 0])
    with pytest.raises(parity.ParityError):
        parity.check_indices(bad, s, np.full_like(gap, 1.0), k)
    with pytest.raises(parity.ParityError):
        parity.check_indices(bad, s, np.zeros_like(gap), k)


def test_checker_rejects_duplicate_and_order():
    s, idx, gap, k, _ = _case()
    dup = idx.copy()
    dup[0, 0, 1] = dup[0, 0, 0]
    with pytest.raises(parity.ParityError):
        parity.check_indices(dup, s, gap, k)
    rev = idx[:, :, ::-1].copy()
    with pytest.raises(parity.ParityError):
        parity.check_indices(rev, s, gap, k)


def test_checker_rejects_attention_error():
    ref = np.random.default_rng(1).standard_normal((2, 4, 16))
    out = ref.copy()
    parity.check_attention(out, None, ref, None)
    out[1, 2, 3] += 3e-3
    with pytest.raises(parity.ParityError):
        parity.check_attention(out, None, ref, None)


def test_checker_rejects_prune_change():
    ref = np.arange(10)[None]
    parity.check_prune(ref.copy(), ref)
    bad = ref.copy()
    bad[0, 4] = 11
    with pytest.raises(parity.ParityError):
        parity.check_prune(bad, ref)


@pytest.mark.parametrize("case,status", [("P0", 1), ("P9", 1), ("rank", 1), ("epoch0", 1),
                                         ("null_peers", 1), ("shard", 2)])
def test_push_host_validation(svl, case, status):
    """svl_sparse_decode_attn_push rejects bad multi-GPU arguments on the host
    (SURVEY.md 8(b) b6/b7), before any launch."""
    L = svl.lib()
    P_ = 0x10000
    peers = (ctypes.c_void_p * 2)(P_, P_)
    args = dict(q=P_, B=1, H=28, Hkv=4, d=128, K=_kv(), V=_kv(), sp=svl.svl_span(10, 60, P_),
                idx=P_, k=10, flags=0, scale=0.088, out=P_, lse=None,
                po=ctypes.cast(peers, ctypes.c_void_p), pf=ctypes.cast(peers, ctypes.c_void_p),
                rank=0, P=2, epoch=1, b0=0, h0=0, Bt=1, Ht=56, ws=P_, wsb=1 << 20, st=None)
    if case == "P0":
        args["P"] = 0
    elif case == "P9":
        args["P"] = 9
    elif case == "rank":
        args["rank"] = 2
    elif case == "epoch0":
        args["epoch"] = 0
    elif case == "null_peers":
        args["po"] = None
    elif case == "shard":
        args["h0"] = 40          # 40 + 28 > 56
    rc = L.svl_sparse_decode_attn_push(*args.values())
    assert rc == status, (rc, L.svl_last_error_message())
    rc = L.svl_wait_flags(P_, 0 if case == "P0" else 2, 0 if case == "epoch0" else 1, None, None)
    assert rc == 1


@pytest.mark.parametrize("case,status", [
    ("small_packed", 2), ("k_gt_nv", 1), ("bad_flags", 1), ("null_idx", 1), ("bad_d", 5), ("null_ws", 4),
    ("cap_mismatch", 2)])
def test_pack_host_validation(svl, case, status):
    """svl_pack_kv: host-checkable errors return before any launch."""
    L = svl.lib()
    P = 0x10000
    sv = svl_mod()
    # source capacity 100, span [10, 70): packed capacity needed = 10 + k + 30
    args = dict(K=_kv(), V=_kv(), B=1, Hkv=4, d=128, sp=sv.svl_span(10, 60, P), idx=P, k=20, flags=0,
                Kp=_kv(cap=60), Vp=_kv(cap=60), ws=P, wsb=1 << 20, st=None)
    if case == "small_packed":
        args["Kp"], args["Vp"] = _kv(cap=59), _kv(cap=59)
    elif case == "k_gt_nv":
        args["k"] = 61
    elif case == "bad_flags":
        args["flags"] = 4
    elif case == "null_idx":
        args["idx"] = None
    elif case == "bad_d":
        args["d"] = 96
        for key in ("K", "V", "Kp", "Vp"):
            args[key] = _kv(cap=100 if key in ("K", "V") else 60, d=96)
    elif case == "null_ws":
        args["ws"] = None
    elif case == "cap_mismatch":
        args["Vp"] = _kv(cap=61)
    rc = L.svl_pack_kv(*args.values())
    assert rc == status, (rc, L.svl_last_error_message())


@pytest.mark.gpu
def test_fresh_plan_multi_wave_rule():
    """The fresh-step planner (svl_fresh_decode_plan, host only): one wave of 16-CTA clusters,
    or up to three over slices >= 1536 rows; two calls beyond (or over short slices).  Needs
    the device's co-resident cluster count, so it is skipped without a GPU."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs the device's cluster occupancy")
    from paper_2510_17777_b200 import svl
    lib = svl.lib()
    plan = lambda B, nv: lib.svl_fresh_decode_plan(B, 28, 4, 128, nv, nv + 1024, 0)
    assert plan(1, 32768) == 1 and plan(3, 32768) == 1 and plan(5, 32768) == 1
    assert plan(8, 16384) == 0 and plan(16, 65536) == 0
