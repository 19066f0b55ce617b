"""Parity rules of SURVEY.md 8(c) c6.

* retrieve indices: per unit, with the oracle's rel_gap = (S_(k)-S_(k+1))/|S_(k)|:
  - rel_gap > 1e-4  -> GPU set == oracle set, bit-exact;
  - otherwise the GPU set must contain every j with S_j > S_(k)(1+1e-4) and be
    a subset of {j : S_j >= S_(k)(1-1e-4)};
  - always |set| = k, ascending, unique, in range.
* attention: per (b, h): max|out-ref| <= 2e-3 and ||out-ref||/||ref|| <= 1e-2;
  |lse - lse_ref| <= 1e-3.
* prune: bit-exact.
* salience: max|sal - ref| <= 1e-5 * max|ref| + 1e-7.
"""
import numpy as np

GAP = 1e-4
ATT_ABS, ATT_REL, LSE_ABS = 2e-3, 1e-2, 1e-3
SAL_REL, SAL_ABS = 1e-5, 1e-7


class ParityError(AssertionError):
    pass


def check_indices(gpu_idx, scores, rel_gap, k):
    """gpu_idx [B][U][k] int; scores [B][U][N] float64 oracle; rel_gap [B][U].
    Returns the fraction of units in the strict (bit-exact) regime."""
    gpu_idx = np.asarray(gpu_idx)
    scores = np.asarray(scores)
    B, U, N = scores.shape
    strict = 0
    for b in range(B):
        for u in range(U):
            g = gpu_idx[b, u]
            if len(g) != k:
                raise ParityError(f"unit ({b},{u}): |set| {len(g)} != k {k}")
            if k == 0:
                strict += 1
                continue
            if np.any(g < 0) or np.any(g >= N):
                raise ParityError(f"unit ({b},{u}): index out of range")
            if np.any(np.diff(g) <= 0):
                raise ParityError(f"unit ({b},{u}): not strictly ascending")
            s = scores[b, u]
            order = np.lexsort((np.arange(N), -s))
            ref = np.sort(order[:k])
            if rel_gap[b, u] > GAP:
                strict += 1
                if not np.array_equal(g, ref):
                    bad = np.setdiff1d(g, ref)[:5]
                    raise ParityError(f"unit ({b},{u}): set differs (gap {rel_gap[b, u]:.3g}), "
                                      f"extra {bad.tolist()}")
            else:
                sk = s[order[k - 1]]
                must = np.nonzero(s > sk * (1 + GAP))[0]
                may = s >= sk * (1 - GAP)
                if not np.all(np.isin(must, g)):
                    raise ParityError(f"unit ({b},{u}): misses a clearly-selected row")
                if not np.all(may[g]):
                    raise ParityError(f"unit ({b},{u}): selects a clearly-unselected row")
    return strict / float(B * U)


def check_attention(out, lse, ref_out, ref_lse):
    out = np.asarray(out, np.float64)
    ref_out = np.asarray(ref_out, np.float64)
    err = np.abs(out - ref_out)
    mx = err.max() if err.size else 0.0
    if mx > ATT_ABS:
        i = np.unravel_index(np.argmax(err), err.shape)
        raise ParityError(f"attention max-abs {mx:.3g} > {ATT_ABS} at {i}")
    num = np.linalg.norm((out - ref_out).reshape(-1, out.shape[-1]), axis=-1)
    den = np.linalg.norm(ref_out.reshape(-1, out.shape[-1]), axis=-1)
    rel = num / np.maximum(den, 1e-30)
    if rel.max() > ATT_REL:
        raise ParityError(f"attention relative {rel.max():.3g} > {ATT_REL}")
    if lse is not None:
        le = np.abs(np.asarray(lse, np.float64) - np.asarray(ref_lse, np.float64)).max()
        if le > LSE_ABS:
            raise ParityError(f"lse max-abs {le:.3g} > {LSE_ABS}")
    return mx, rel.max()


def check_prune(gpu, ref):
    gpu, ref = np.asarray(gpu), np.asarray(ref)
    if gpu.shape != ref.shape or not np.array_equal(gpu, ref):
        diff = np.nonzero(gpu != ref) if gpu.shape == ref.shape else "shape"
        raise ParityError(f"prune indices differ: {diff}")


def check_salience(sal, ref):
    sal, ref = np.asarray(sal, np.float64), np.asarray(ref, np.float64)
    tol = SAL_REL * np.abs(ref).max() + SAL_ABS
    e = np.abs(sal - ref).max()
    if e > tol:
        raise ParityError(f"salience max-abs {e:.3g} > {tol:.3g}")
    return e
