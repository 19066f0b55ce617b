#!/usr/bin/env python
"""bench.py -- SparseVILA decode-stage hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {svl,reference}]

N = 1 (default): the headline.  Step = one fresh-retrieval decode step of a
28-layer stack (NVILA-8B / Qwen2-7B depth) on the long-video workload
(BASELINE.json configs[2]: 32768 retained visual tokens, 512 + 256 text rows at
the last of 256 generated tokens, k = keep_budget(32768, 0.90) = 3277, batch
1, 28 q / 4 KV heads, d = 128): per layer ONE svl_fresh_decode_step (retrieve
a1-a3 + sparse decode a4-a5 fused; fresh_kernel) through the C ABI, replayed
as one CUDA graph.  28 distinct layer KV caches (1.9 GB) rotate, so the
working set is > L2 every step.

N > 1: `python bench.py --gpus N` re-launches itself under torch.distributed.run
(one rank per GPU, NCCL).  Default there: the throughput-sweep config
(BASELINE.json configs[4]: B 16, 65536 visual, k 6554) sharded over (batch x KV
head) (sharding.plan), one svl_fresh_decode_step per layer per rank and one
NCCL all-gather of the fp32 head outputs per layer, captured in the same CUDA
graph: strong scaling; rank 0 also times the unsharded step on its GPU alone,
so the line carries E(P) = T(1) / (P T(P)) with and without the gather.
--mode replicas: every rank serves its own long-video request (weak scaling).

value  = algorithmic HBM bytes of the step (scored visual
         K + selected K/V + text K/V once + q + out + idx) / step time, summed
         over ranks.
e2e    = the same through the public API with host buffers: per step the
         new token's q and K/V rows go H2D from pinned memory, the graph
         replays, and the attention outputs come back D2H.
--impl reference = the fp64 CPU oracle (oracle/), the paper-method baseline
         of this tier, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LAYERS = 28
WORKLOAD = "long-video"
ROUND_STEPS = 256  # decode steps per retrieval round (BASELINE.json long-video: 256 generated tokens)
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def step_bytes(wl, n_q=1):
    """Algorithmic bytes of one layer's fresh-retrieval step:
    scored visual K + selected K,V + text K,V (text K counted once) + q + out + idx."""
    T = wl.vb + wl.t_after                   # text rows attended at this step
    row = wl.d * 2
    kvis = wl.B * wl.Hkv * wl.nv * row
    sel = wl.B * wl.Hkv * wl.k * 2 * row
    text = wl.B * wl.Hkv * T * 2 * row
    q = wl.B * n_q * wl.H * row
    out = wl.B * wl.H * wl.d * 4
    idx = wl.B * wl.Hkv * wl.k * 4
    return {"score": kvis + wl.B * wl.Hkv * T * row + q,   # what the scoring kernel must read
            # what the fused fresh-step kernel must move: K streamed once (visual +
            # text; the decode reuses the retrieval logits), kept V + text V, q, out, idx
            "fused": kvis + wl.B * wl.Hkv * T * row + sel // 2 + text // 2 + q + out + idx,
            "total": kvis + sel + text + q + out + idx,
            # steady step: the sparse decode alone (selected + text K and V, q in, out + idx)
            "decode": sel + text + q + out + idx}


def kv_cache_bytes(entries, layers, kv_heads, d, elem_bytes):
    """SPEC.md:331 cache_stats byte accounting: entries * 2 (K and V) * d * heads * layers * width."""
    return entries * 2 * d * kv_heads * layers * elem_bytes


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.strip().splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def quantile(xs, q):
    ys = sorted(xs)
    if not ys:
        return None
    pos = q * (len(ys) - 1)
    lo = int(pos)
    hi = min(lo + 1, len(ys) - 1)
    return ys[lo] + (ys[hi] - ys[lo]) * (pos - lo)


def replay_times(g, n):
    """ms of each of n graph replays (CUDA events around every replay)."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def cold_layer_us(fn, n=30):
    """Median us of one launch of fn() after a 2 x L2 write (cold L2, nothing in flight)."""
    import torch
    flush = torch.empty(2 * 126 * 2 ** 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(n):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    del flush
    return statistics.median(ts)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- CPU oracle


def cpu_oracle_sample(wl, budget_s=12.0, nthreads=None):
    """Time the fp64 oracle (as it stands) on whole layers of the workload
    until ~budget_s of CPU work; returns (bytes/s, layers, threads, seconds)."""
    import oracle
    import torch
    from paper_2510_17777_b200 import inputs as gen
    nthreads = nthreads or os.cpu_count() or 1
    x = gen.make_decode_inputs(wl, seed=0)
    nb = step_bytes(wl)["total"]
    layers, t_total = 0, 0.0
    while t_total < budget_s and layers < LAYERS:
        t0 = time.perf_counter()
        idx, _, _ = oracle.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k,
                                    nthreads=nthreads)
        oracle.sparse_decode(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx,
                             nthreads=nthreads)
        t_total += time.perf_counter() - t0
        layers += 1
    _ = torch
    return nb * layers / t_total, layers, nthreads, t_total


def kernel_src_sha(names=("fused.cu", "select_fast.cuh", "select_push.cuh", "common.cuh", "kernels.h")):
    import hashlib
    h = hashlib.sha256()
    for n in names:
        h.update(open(os.path.join(ROOT, "paper_2510_17777_b200", "csrc", n), "rb").read())
    return h.hexdigest()[:16]


def fresh_traffic():
    """dram bytes per fresh_kernel launch from the committed ncu capture, only while that
    capture's kernel source hash matches the current source (else null)."""
    tp = os.path.join(ROOT, "profiles", "ncu_fresh_traffic.json")
    try:
        d = json.load(open(tp))
    except (OSError, ValueError):
        return None, None
    if d.get("src_sha") != kernel_src_sha():
        return None, "stale: profiles/ncu_fresh_traffic.json was captured from another fresh_kernel source"
    return d.get("dram_bytes_per_launch"), d.get("source")


def config_rows(graph_of, timed):
    """SURVEY.md 8(d) d2 rows beside the headline: per config the fresh step and the steady
    decode per layer (CUDA graphs over rotating layer caches larger than L2) and the
    per-round amortised step."""
    import torch

    from paper_2510_17777_b200 import inputs as gen
    from paper_2510_17777_b200 import svl
    out = {}
    for name, nrot, round_len in (("nvila-4k", 77, ROUND_STEPS), ("multi-turn", LAYERS, 250)):
        wl = gen.CONFIGS[name]
        xs = [gen.make_decode_inputs(wl, seed=3000 + l, device="cuda") for l in range(nrot)]
        idx = [torch.empty(wl.B, wl.Hkv, wl.k, dtype=torch.int32, device="cuda") for _ in range(nrot)]
        outs = [torch.empty(wl.B, wl.H, wl.d, device="cuda") for _ in range(nrot)]
        wsf, wsd = svl.Workspace(), svl.Workspace()
        wsf.get(svl.fresh_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))
        wsd.get(svl.sparse_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))
        g_f = graph_of(lambda: [svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k,
                                                      idx_out=i, out=o, ws=wsf) for x, i, o in zip(xs, idx, outs)])
        # steady decode: the selection of the round's fresh step (another graph) -- static
        g_d = graph_of(lambda: [svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, i,
                                                       flags=svl.SVL_DECODE_STATIC_PREFIX, out=o, ws=wsd)
                                for x, i, o in zip(xs, idx, outs)])
        f_us = timed(g_f, 100, 10) * 1e3 / nrot
        d_us = timed(g_d, 100, 10) * 1e3 / nrot
        b = step_bytes(wl)
        am = (f_us + (round_len - 1) * d_us) / round_len
        out[name] = {"B": wl.B, "visual_tokens": wl.nv, "k": wl.k,
                     "fresh_us_per_layer": f_us, "fresh_GB_s": b["total"] / (f_us * 1e-6) / 1e9,
                     "fresh_path": "fused" if svl.fresh_uses_fused(wl.B, wl.H, wl.Hkv, wl.d, wl.nv, wl.capacity)
                     else "two calls",
                     "steady_us_per_layer": d_us, "steady_GB_s": b["decode"] / (d_us * 1e-6) / 1e9,
                     "amortized_us_per_layer": am,
                     "amortized_what": f"(1 fresh + {round_len - 1} steady) / {round_len} per round",
                     "tokens_per_s_28_layers": wl.B / (am * 1e-6 * LAYERS),
                     "rotating_layers": nrot}
        del xs, g_f, g_d
    return out


def page_row(graph_of, timed, page=16):
    """retrieval on page summaries (Quest-style, reading A22) on the
    long-video cache: the summaries are built once per retained cache; per decode step the
    page scores + top-k pages + the decode over the kept pages' rows.  Recall = the share of
    the exact fresh step's kept rows that the kept pages contain; err = max |out - exact out|."""
    import torch

    from paper_2510_17777_b200 import inputs as gen
    from paper_2510_17777_b200 import svl
    wl = gen.CONFIGS[WORKLOAD]
    nl = LAYERS
    xs = [gen.make_decode_inputs(wl, seed=5000 + l, device="cuda") for l in range(nl)]
    kp = wl.k // page
    summ = [svl.page_summary(x["K"], wl.vb, wl.nv, page) for x in xs]
    pidx = [torch.empty(wl.B, wl.Hkv, kp, dtype=torch.int32, device="cuda") for _ in range(nl)]
    rows = [torch.empty(wl.B, wl.Hkv, kp * page, dtype=torch.int32, device="cuda") for _ in range(nl)]
    outs = [torch.empty(wl.B, wl.H, wl.d, device="cuda") for _ in range(nl)]
    wsr, wsd, wss = svl.Workspace(), svl.Workspace(), svl.Workspace()
    wsd.get(svl.sparse_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, kp * page, wl.nv, wl.capacity))

    def retr(l):
        svl.retrieve_pages(xs[l]["q"], summ[l][0], summ[l][1], page, kp, page_idx_out=pidx[l], row_idx_out=rows[l],
                           ws=wsr)

    def dec(l):
        svl.sparse_decode_attn(xs[l]["q_dec"], xs[l]["K"], xs[l]["V"], xs[l]["seq_len"], wl.vb, wl.nv, rows[l],
                               out=outs[l], ws=wsd)

    g_step = graph_of(lambda: [(retr(l), dec(l)) for l in range(nl)])
    g_retr = graph_of(lambda: [retr(l) for l in range(nl)])
    g_sum = graph_of(lambda: [svl.page_summary(xs[l]["K"], wl.vb, wl.nv, page, kmax=summ[l][0], kmin=summ[l][1],
                                               ws=wss) for l in range(nl)])
    step_us = timed(g_step, 200, 10) * 1e3 / nl
    retr_us = timed(g_retr, 200, 10) * 1e3 / nl
    sum_us = timed(g_sum, 50, 5) * 1e3 / nl
    # quality vs the exact fresh step (same layer 0 inputs)
    ex_out, ex_idx = svl.fresh_decode_step(xs[0]["q_dec"], xs[0]["K"], xs[0]["V"], xs[0]["seq_len"], wl.vb, wl.nv,
                                           wl.k)
    g_step.replay()
    torch.cuda.synchronize()
    recall = []
    for G in range(wl.Hkv):
        kept = set(rows[0][0, G].tolist())
        ex = ex_idx[0, G].tolist()
        recall.append(sum(1 for j in ex if j in kept) / len(ex))
    err = (outs[0] - ex_out).abs().max().item()
    b = step_bytes(wl)
    row = wl.d * 2
    scored = wl.B * wl.Hkv * (wl.nv // page) * 2 * row
    dec_bytes = b["decode"] - wl.B * wl.Hkv * wl.k * 2 * row + wl.B * wl.Hkv * kp * page * 2 * row
    return {"what": "svl_retrieve_pages (page bounds, softmax over pages, top-k pages) + svl_sparse_decode_attn over "
                    "the kept pages' rows, long-video, 28-layer graph (SURVEY.md 8(f) f2(ii), reading A22)",
            "page": page, "k_pages": kp, "rows_kept": kp * page,
            "us_per_layer": step_us, "retrieve_us_per_layer": retr_us,
            "summary_build_us_per_layer": sum_us, "summary_build_when": "once per retained cache (prefill / round)",
            "scored_bytes_per_layer": scored, "exact_scored_bytes_per_layer": wl.B * wl.Hkv * wl.nv * row,
            "step_bytes_per_layer": scored + dec_bytes,
            "GB_s": (scored + dec_bytes) / (step_us * 1e-6) / 1e9,
            "recall_vs_exact_topk": recall, "max_abs_out_vs_exact_fresh_step": err}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    """The reference arm of this tier: the fp64 CPU oracle, as it stands, on the
    box's host cores.  One step = `sample` whole layers of the long-video step
    (retrieve + sparse decode), sized after timing one layer so that the whole
    --steps K --warmup W run ends within ~2 minutes; ms_per_step is the measured
    time of that step (no extrapolation) and config.layers says how many layers
    a step holds."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2510_17777_b200 import inputs as gen
    wl = gen.CONFIGS[WORKLOAD]
    per_layer = step_bytes(wl)["total"]
    import oracle
    x = gen.make_decode_inputs(wl, seed=0)
    nth = os.cpu_count() or 1

    def layer():
        idx, _, _ = oracle.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, nthreads=nth)
        oracle.sparse_decode(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx, nthreads=nth)

    t0 = time.perf_counter()
    layer()
    t_layer = time.perf_counter() - t0
    sample = int(max(1, min(LAYERS, 120.0 / max(1, args.steps + args.warmup) / max(t_layer, 1e-6))))
    for _ in range(args.warmup):
        for _ in range(sample):
            layer()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(sample):
            layer()
    dt = time.perf_counter() - t0
    ms_step = dt * 1e3 / args.steps
    value = per_layer * sample / (ms_step * 1e-3) / 1e9
    cfg = config_dict(wl)
    cfg["layers"] = sample
    cfg["workload"] = f"{WORKLOAD}: {sample}-layer sample of the {LAYERS}-layer fresh-retrieval decode step"
    line = {
        "impl": "reference", "metric": "decode step HBM GB/s (retrieve+sparse attn) @32k visual tok",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": nth, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{sample} of {LAYERS} layers per step, measured (fp64 C oracle, "
                                   f"OpenMP over the (b, KV group) units)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def config_dict(wl):
    return {"workload": f"{WORKLOAD}: {LAYERS}-layer fresh-retrieval decode step",
            "B": wl.B, "H": wl.H, "Hkv": wl.Hkv, "d": wl.d, "visual_tokens": wl.nv,
            "text_rows": wl.vb + wl.t_after, "k": wl.k, "decode_sparsity": 0.90, "layers": LAYERS,
            "l2": "inputs > L2: 28 rotating layer KV caches (1.9 GB) per step"}


# ---------------------------------------------------------------- GPU arm


def fused_gather_timing(wl, sp, loc, world, rank, dev, steps):
    """Per layer: svl_retrieve on the rank's slice, then svl_sparse_decode_attn_push into
    every rank's gathered [B][H][d] buffer (symmetric memory across processes), then
    svl_wait_flags for every producer's epoch.  Returns ms per 28-layer step (max over
    ranks) or the reason it could not run."""
    import torch
    import torch.distributed as dist

    from paper_2510_17777_b200 import svl
    try:
        if world > 1:
            import torch.distributed._symmetric_memory as symm_mem
            bufs, flags = [], []
            for _ in range(SHARD_ROT):
                t = symm_mem.empty(wl.B * wl.H * wl.d, dtype=torch.float32, device=dev)
                h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
                bufs.append([h.get_buffer(r, (wl.B, wl.H, wl.d), torch.float32) for r in range(world)])
            tf = symm_mem.empty(world, dtype=torch.int32, device=dev)
            tf.zero_()
            hf = symm_mem.rendezvous(tf, dist.group.WORLD.group_name)
            flags = [hf.get_buffer(r, (world,), torch.int32) for r in range(world)]
            dist.barrier()
        else:
            bufs = [[torch.empty(wl.B, wl.H, wl.d, device=dev)] for _ in range(SHARD_ROT)]
            tf = torch.zeros(1, dtype=torch.int32, device=dev)
            flags = [tf]
    except Exception as e:  # noqa: BLE001 -- report, do not fail the bench line
        return {"unavailable": f"symmetric memory: {type(e).__name__}: {str(e)[:120]}"}
    Hkvl = sp.kv1 - sp.kv0
    ws = svl.Workspace(dev)
    wsw = svl.Workspace(dev)
    idx = torch.empty(sp.B_local, Hkvl, wl.k, dtype=torch.int32, device=dev)
    epoch = [0]

    def step():
        for l in range(LAYERS):
            r = l % SHARD_ROT
            ql, Kl, Vl, sl = loc[r]
            epoch[0] += 1
            svl.retrieve(ql.unsqueeze(1), Kl, sl, wl.vb, wl.nv, wl.k, idx_out=idx, ws=ws)
            svl.sparse_decode_attn_push(ql, Kl, Vl, sl, wl.vb, wl.nv, idx, bufs[r], flags, rank, epoch[0],
                                        sp.b0, sp.kv0 * sp.g, ws=ws)
            svl.wait_flags(tf, epoch[0], ws=wsw)

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    timeouts = bool(wsw.flags() & svl.SVL_DEVFLAG_WAIT_TIMEOUT)
    return {"ms_per_step": ms, "steps": steps, "wait_timeouts": timeouts,
            "how": "eager: svl_retrieve + svl_sparse_decode_attn_push (peer stores into symmetric memory) + "
                   "svl_wait_flags per layer"}


SHARD_ROT = 4  # rotating layer caches of the sharded runs (the 28-layer step cycles through them)


def run_sharded(args, cfg_name):
    """one batch (the throughput sweep by default) sharded over
    (batch x KV head) (sharding.plan: P_h = gcd(P, Hkv), P_b = P / P_h), one
    svl_fresh_decode_step per layer per rank on its slice of every layer's cache,
    then one NCCL all_gather_into_tensor of the fp32 head outputs per layer (the
    harness's exchange, north star), permuted into [B][H][d] -- all captured in
    one CUDA graph per 28-layer step.  Strong scaling: the total work is fixed.
    Rank 0 also times the same 28-layer step unsharded on its GPU alone (T(1)), so
    the line carries E(P) = T(1) / (P T(P)) with and without the gather."""
    import torch
    import torch.distributed as dist

    from paper_2510_17777_b200 import inputs as gen
    from paper_2510_17777_b200 import sharding, svl

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    svl.lib()
    wl = gen.CONFIGS[cfg_name]
    sp = sharding.plan(wl.B, wl.H, wl.Hkv, world, rank)
    # every rank generates the same global layers and keeps views of its slice (the
    # sharded outputs can then be checked against the unsharded run); ~1.3 GB per sweep layer
    xs = [gen.make_decode_inputs(wl, seed=7000 + l, device=dev) for l in range(SHARD_ROT)]
    loc = [sharding.local_inputs(sp, x["q_dec"], x["K"], x["V"], x["seq_len"]) for x in xs]
    Bl, Hl, Hkvl = sp.B_local, sp.H_local, sp.kv1 - sp.kv0
    ws = svl.Workspace(dev)
    ws.get(svl.fresh_decode_workspace_size(Bl, Hl, Hkvl, wl.d, wl.k, wl.nv, wl.capacity))
    outs = [torch.empty(Bl, Hl, wl.d, device=dev) for _ in range(SHARD_ROT)]
    idxs = [torch.empty(Bl, Hkvl, wl.k, dtype=torch.int32, device=dev) for _ in range(SHARD_ROT)]
    gbuf = [torch.empty(world * Bl * Hl * wl.d, device=dev) for _ in range(SHARD_ROT)]
    full = [torch.empty(wl.B, wl.H, wl.d, device=dev) for _ in range(SHARD_ROT)]
    plans = [sharding.plan(wl.B, wl.H, wl.Hkv, world, r) for r in range(world)]
    # permutation of the gathered rank blocks into [B][H][d] (a gather by index: graph-safe)
    perm = torch.empty(wl.B, wl.H, dtype=torch.int64)
    for r, pr in enumerate(plans):
        bb, hh = torch.meshgrid(torch.arange(pr.B_local), torch.arange(pr.H_local), indexing="ij")
        perm[pr.b0:pr.b1, pr.kv0 * pr.g:pr.kv1 * pr.g] = r * pr.B_local * pr.H_local + bb * pr.H_local + hh
    perm = perm.view(-1).to(dev)

    def layer(l, gather):
        r = l % SHARD_ROT
        ql, Kl, Vl, sl = loc[r]
        svl.fresh_decode_step(ql, Kl, Vl, sl, wl.vb, wl.nv, wl.k, idx_out=idxs[r], out=outs[r], ws=ws)
        if gather:
            if world > 1:
                dist.all_gather_into_tensor(gbuf[r], outs[r].view(-1))
            else:
                gbuf[r].copy_(outs[r].view(-1))
            torch.index_select(gbuf[r].view(-1, wl.d), 0, perm, out=full[r].view(-1, wl.d))

    def graph_of(fn):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(st):
            with torch.cuda.graph(g, stream=st):
                fn()
        torch.cuda.synchronize()
        return g

    def timed(g, steps, warmup):
        for _ in range(warmup):
            g.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

    steps = max(5, min(args.steps, 200))
    warm = max(3, min(args.warmup, 20))
    # ---- T(1): rank 0 alone, the unsharded step (same layers, same 28-layer structure)
    t1 = None
    ref_out = None
    if rank == 0:
        ws1 = svl.Workspace(dev)
        ws1.get(svl.fresh_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))
        o1 = [torch.empty(wl.B, wl.H, wl.d, device=dev) for _ in range(SHARD_ROT)]
        i1 = [torch.empty(wl.B, wl.Hkv, wl.k, dtype=torch.int32, device=dev) for _ in range(SHARD_ROT)]

        def one_gpu():
            for l in range(LAYERS):
                r = l % SHARD_ROT
                svl.fresh_decode_step(xs[r]["q_dec"], xs[r]["K"], xs[r]["V"], xs[r]["seq_len"], wl.vb, wl.nv,
                                      wl.k, idx_out=i1[r], out=o1[r], ws=ws1)
        g1 = graph_of(one_gpu)
        for _ in range(warm):
            g1.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            g1.replay()
        e1.record()
        torch.cuda.synchronize()
        t1 = e0.elapsed_time(e1) / steps
        ref_out = o1[(LAYERS - 1) % SHARD_ROT].clone()
        del g1, o1, i1, ws1
    if world > 1:
        dist.barrier()
    # ---- T(P): the sharded step with and without the gather
    g_full = graph_of(lambda: [layer(l, True) for l in range(LAYERS)])
    g_comp = graph_of(lambda: [layer(l, False) for l in range(LAYERS)])
    with ClockSampler(local) as clk:
        ms = timed(g_full, steps, warm)
    ms_c = timed(g_comp, steps, warm)
    # the gathered output equals the unsharded one (per-unit split counts differ between a
    # shard and the whole batch, so within the attention tolerance, not bitwise)
    check = None
    if rank == 0:
        g_full.replay()
        torch.cuda.synchronize()
        got = full[(LAYERS - 1) % SHARD_ROT]
        check = {"max_abs_vs_unsharded": float((got - ref_out).abs().max().item())}
    # ---- --fused-gather: the exchange folded into the decode kernel (svl_sparse_decode_attn_push
    # stores every output element into each rank's symmetric-memory buffer, then raises the
    # rank's epoch flag; svl_wait_flags is the consumer).  Eager launches (the epoch is a
    # call argument, so a replayed graph would reuse it).
    fused = None
    if args.fused_gather:
        fused = fused_gather_timing(wl, sp, loc, world, rank, dev, steps=max(3, steps // 10))
    # ---- e2e through the public API: per step the ranks' q slices H2D (pinned), the graph,
    # the gathered outputs D2H
    q_host = [loc[r][0].cpu().pin_memory() for r in range(SHARD_ROT)]
    out_host = torch.empty(SHARD_ROT, wl.B, wl.H, wl.d).pin_memory()

    def e2e_once():
        for r in range(SHARD_ROT):
            loc[r][0].copy_(q_host[r], non_blocking=True)
        g_full.replay()
        for r in range(SHARD_ROT):
            out_host[r].copy_(full[r], non_blocking=True)
        torch.cuda.current_stream().synchronize()

    for _ in range(3):
        e2e_once()
    if world > 1:
        dist.barrier()
    n_e2e = max(5, steps // 4)
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        e2e_once()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / n_e2e
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
    total = step_bytes(wl)["total"] * LAYERS
    nccl = {"backend": dist.get_backend() if world > 1 else None, "nranks": world,
            "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if world > 1 else None,
            "gather_bytes_per_layer_per_rank": Bl * Hl * wl.d * 4}
    if rank == 0:
        line = {
            "metric": f"decode step HBM GB/s (retrieve+sparse attn), {cfg_name} batch head-sharded",
            "value": total / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world, "steps": steps,
            "warmup": warm, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded generator)",
            "config": {"workload": f"{cfg_name}: B {wl.B}, {wl.nv} visual, k {wl.k}, {LAYERS} layers "
                                   f"({SHARD_ROT} rotating caches), (batch x KV-head) shards + NCCL "
                                   f"all-gather of head outputs per layer",
                       "P_b": sp.P_b, "P_h": sp.P_h, "B_local": Bl, "kv_heads_local": Hkvl,
                       "l2": "inputs > L2 (rotating layer caches)"},
            "us_per_layer": ms * 1e3 / LAYERS,
            "compute_only": {"ms_per_step": ms_c, "GB_s": total / (ms_c * 1e-3) / 1e9},
            "one_gpu": {"ms_per_step": t1, "GB_s": total / (t1 * 1e-3) / 1e9} if t1 else None,
            "E_strong": (t1 / (world * ms)) if t1 else None,
            "E_strong_compute_only": (t1 / (world * ms_c)) if t1 else None,
            "E_definition": "T(1) / (P T(P)), T(1) = the unsharded step on rank 0's GPU in this run (SURVEY 8(e) e5)",
            "correctness": check,
            "fused_gather": fused,
            "collective": nccl,
            "e2e": {"value": total / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": sum(int(q.numel()) * 2 for q in q_host),
                    "d2h_bytes_per_step": int(out_host.numel()) * 4},
            "gpu_launches": LAYERS * steps * (1 if svl.fresh_uses_fused(Bl, Hl, Hkvl, wl.d, wl.nv, wl.capacity)
                                               else 3),
            "clocks": clk.summary()}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_seq_split(args):
    """ONE long-video request (B = 1) over P GPUs: P_h =
    gcd(P, Hkv) KV-head groups x P_s = P / P_h sequence shards (8 GPUs: 4 x 2).  Per layer
    every rank runs the sequence-split fresh step on its shard view (seqpar.py: partial LSE,
    LSE exchange, scores exchange + global top-k, padded decode, partial exchange + merge;
    NCCL all-gathers inside the sequence group) and the head outputs are all-gathered over
    the world, all in one CUDA graph.  Strong scaling vs the fused step on one GPU."""
    import math as _m

    import torch
    import torch.distributed as dist

    from paper_2510_17777_b200 import inputs as gen
    from paper_2510_17777_b200 import seqpar, svl

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = gen.CONFIGS[WORKLOAD]
    P_h = _m.gcd(world, wl.Hkv)
    P_s = world // P_h
    hg, s = rank % P_h, rank // P_h
    seq_groups = [list(range(h, world, P_h)) for h in range(P_h)]
    groups = [dist.new_group(r) for r in seq_groups] if world > 1 else [None] * P_h
    my_group = groups[hg]
    kv0, kv1 = hg * wl.Hkv // P_h, (hg + 1) * wl.Hkv // P_h
    h0, h1 = kv0 * wl.g, kv1 * wl.g
    xs = [gen.make_decode_inputs(wl, seed=8000 + l, device=dev) for l in range(SHARD_ROT)]
    states = [seqpar.ShardState(x["q_dec"][:, h0:h1].contiguous(), x["K"][:, kv0:kv1], x["V"][:, kv0:kv1],
                                x["seq_len"], wl.vb, wl.nv, wl.k, P_s, s) for x in xs]
    full = [torch.empty(world, wl.B, h1 - h0, wl.d, device=dev) for _ in range(SHARD_ROT)]

    def gather_seq(t):
        if P_s == 1:
            return t.unsqueeze(0)
        buf = t.new_empty((P_s,) + tuple(t.shape))
        dist.all_gather_into_tensor(buf, t.contiguous(), group=my_group)
        return buf

    def step():
        for l in range(LAYERS):
            r = l % SHARD_ROT
            out, _ = seqpar.distributed_step(states[r], my_group, gather=gather_seq)
            if world > 1:
                dist.all_gather_into_tensor(full[r], out)
            else:
                full[r][0].copy_(out)

    def graph_of(fn):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(st):
            with torch.cuda.graph(g, stream=st):
                fn()
        torch.cuda.synchronize()
        return g

    steps = max(5, min(args.steps, 200))
    warm = max(3, min(args.warmup, 20))
    t1 = None
    if rank == 0:
        wsf = svl.Workspace(dev)
        of = [torch.empty(wl.B, wl.H, wl.d, device=dev) for _ in range(SHARD_ROT)]
        g1 = graph_of(lambda: [svl.fresh_decode_step(xs[l % SHARD_ROT]["q_dec"], xs[l % SHARD_ROT]["K"],
                                                     xs[l % SHARD_ROT]["V"], xs[l % SHARD_ROT]["seq_len"], wl.vb,
                                                     wl.nv, wl.k, out=of[l % SHARD_ROT], ws=wsf)
                               for l in range(LAYERS)])
        for _ in range(warm):
            g1.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            g1.replay()
        e1.record()
        torch.cuda.synchronize()
        t1 = e0.elapsed_time(e1) / steps
        del g1
    if world > 1:
        dist.barrier()
    g = graph_of(step)
    for _ in range(warm):
        g.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    total = step_bytes(wl)["total"] * LAYERS
    if rank == 0:
        print(json.dumps({
            "metric": "decode step HBM GB/s (retrieve+sparse attn) @32k visual tok, one request sequence-split",
            "value": total / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded generator)",
            "config": {"workload": f"long-video B=1, {LAYERS} layers ({SHARD_ROT} rotating caches): {P_h} KV-head "
                                   f"groups x {P_s} sequence shards, 3 exchanges per layer in the sequence group + "
                                   "the head-output all-gather", "P_h": P_h, "P_s": P_s},
            "us_per_layer": ms * 1e3 / LAYERS,
            "one_gpu_fused": {"ms_per_step": t1} if t1 else None,
            "E_strong": (t1 / (world * ms)) if t1 else None,
            "gpu_launches": LAYERS * steps * 8, "clocks": clk.summary()}))
    if world > 1:
        dist.destroy_process_group()
    return 0


def free_port():
    import socket
    sck = socket.socket()
    sck.bind(("127.0.0.1", 0))
    port = sck.getsockname()[1]
    sck.close()
    return port


def relaunch(args):
    """--gpus N > 1 without a torch.distributed launcher: re-run this script under
    torch.distributed.run with N ranks (one per GPU), the driver's own launch line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="svl", choices=["svl", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no JSON checks)")
    ap.add_argument("--mode", default="auto",
                    choices=["auto", "headline", "replicas", "sweep-heads", "heads", "seq-split"],
                    help="auto: headline at N = 1, sweep-heads at N > 1; replicas: every rank serves its "
                         "own long-video request (weak); sweep-heads: the B 16 / 64k sweep sharded over "
                         "(batch x KV head) with a per-layer NCCL all-gather of the head outputs (strong); "
                         "heads: the same for the multi-turn batch; seq-split: one long-video request over "
                         "KV-head groups x sequence shards (SURVEY 8(f) f3)")
    ap.add_argument("--fused-gather", action="store_true",
                    help="sweep-heads: replace the NCCL all-gather by svl_sparse_decode_attn_push into "
                         "symmetric-memory peer buffers (eager launches: the epoch is a call argument)")
    ap.add_argument("--launch-check", action="store_true", help="print rank / world and exit (launcher test)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ and args.gpus not in (1, world):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.launch_check:
        # one write(2) per rank: the ranks share the pipe, and print's separate newline write interleaves
        sys.stdout.flush()
        os.write(1, (json.dumps({"launch_check": True, "rank": rank, "world": world, "local_rank": local}) + "\n").encode())
        return 0
    if args.impl == "reference":
        return run_reference(args)
    mode = args.mode if args.mode != "auto" else ("headline" if world == 1 else "sweep-heads")
    if mode == "sweep-heads":
        return run_sharded(args, "sweep")
    if mode == "heads":
        return run_sharded(args, "multi-turn")
    if mode == "seq-split":
        return run_seq_split(args)
    return run_headline(args)


def run_headline(args):
    """N = 1: the headline long-video line (+ companions); N > 1 (--mode replicas):
    every rank serves its own long-video request, weak scaling."""
    import torch
    import torch.distributed as dist

    from paper_2510_17777_b200 import inputs as gen
    from paper_2510_17777_b200 import svl

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    svl.lib()

    wl = gen.CONFIGS[WORKLOAD]
    nbytes = step_bytes(wl)
    # ---- 28 distinct layers (rank-dependent seeds: independent requests per rank)
    Ks, Vs, qs, qds = [], [], [], []
    for layer in range(LAYERS):
        x = gen.make_decode_inputs(wl, seed=1000 * rank + layer, device=dev)
        Ks.append(x["K"])
        Vs.append(x["V"])
        qs.append(x["q"])
        qds.append(x["q_dec"])
        seq = x["seq_len"]
    idxs = [torch.empty(wl.B, wl.Hkv, wl.k, dtype=torch.int32, device=dev) for _ in range(LAYERS)]
    out_all = torch.empty(LAYERS, wl.B, wl.H, wl.d, dtype=torch.float32, device=dev)  # one D2H for e2e
    outs = [out_all[l] for l in range(LAYERS)]
    ws_r, ws_d = svl.Workspace(dev), svl.Workspace(dev)
    ws_r.get(svl.retrieve_workspace_size(wl.B, 1, wl.H, wl.Hkv, wl.d, wl.nv))
    ws_d.get(svl.sparse_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))

    def layer_retrieve(l, flags=0):
        svl.retrieve(qs[l], Ks[l], seq, wl.vb, wl.nv, wl.k, flags=flags, idx_out=idxs[l], ws=ws_r)

    def layer_decode(l, flags=0):
        svl.sparse_decode_attn(qds[l], Ks[l], Vs[l], seq, wl.vb, wl.nv, idxs[l], flags=flags, out=outs[l],
                               ws=ws_d)

    ws_f = svl.Workspace(dev)
    ws_f.get(svl.fresh_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))

    def layer_fresh(l):
        svl.fresh_decode_step(qds[l], Ks[l], Vs[l], seq, wl.vb, wl.nv, wl.k, idx_out=idxs[l],
                              out=outs[l], ws=ws_f)

    def full_step():
        for l in range(LAYERS):
            layer_fresh(l)

    def unfused_step():
        for l in range(LAYERS):
            layer_retrieve(l)
            layer_decode(l)

    def graph_of(fn):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                fn()
        torch.cuda.synchronize()
        return g

    g_step = graph_of(full_step)
    g_unfused = graph_of(unfused_step)
    g_score = graph_of(lambda: [layer_retrieve(l, svl.SVL_RETRIEVE_SCORE_ONLY) for l in range(LAYERS)])
    g_select = graph_of(lambda: [layer_retrieve(l, svl.SVL_RETRIEVE_SELECT_ONLY) for l in range(LAYERS)])
    # steady decode: idxs are the last fresh step's selection, the rows below the current
    # token's were written by earlier steps -- SVL_DECODE_STATIC_PREFIX (their gathers start
    # before the PDL wait); the unfused graph above writes idxs[l] right before
    # layer_decode(l), so it runs without
    g_decode = graph_of(lambda: [layer_decode(l, svl.SVL_DECODE_STATIC_PREFIX) for l in range(LAYERS)])
    g_decode_plain = graph_of(lambda: [layer_decode(l) for l in range(LAYERS)])  # (no early gathers)

    if args.profile:
        for _ in range(max(args.warmup, 1)):
            g_step.replay()
        for _ in range(args.steps):
            g_step.replay()
        torch.cuda.synchronize()
        return 0

    def timed(g, steps, warmup):
        for _ in range(warmup):
            g.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return e0.elapsed_time(e1) / steps  # ms per replay

    # ---- headline: the full 28-layer step, clocks sampled during the timed region
    with ClockSampler(local) as clk:
        ms_step = timed(g_step, args.steps, args.warmup)
    clocks = clk.summary()
    if world > 1:
        t = torch.tensor([ms_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = t.item()
    total_bytes = nbytes["total"] * LAYERS * world
    value = total_bytes / (ms_step * 1e-3) / 1e9
    # per-replay distribution (events around each replay): median / p10 / p90 per step
    dist_ms = replay_times(g_step, min(200, args.steps))
    pct = {"median": statistics.median(dist_ms), "p10": quantile(dist_ms, 0.10),
           "p90": quantile(dist_ms, 0.90), "n": len(dist_ms)}
    # cold single layer: a 2 x L2 write before each launch, events
    # around the one launch only -- no overlap with a neighbouring layer
    cold_fresh_us = cold_layer_us(lambda: layer_fresh(0))
    cold_decode_us = cold_layer_us(lambda: layer_decode(0))

    # ---- breakdown (same stream, CUDA events): score / select / decode graphs
    sub = max(200, args.steps // 4)
    ms_unfused = timed(g_unfused, sub, 10)
    ms_score = timed(g_score, sub, 10)
    ms_select = timed(g_select, sub, 10)
    ms_decode = timed(g_decode, sub, 10)
    ms_decode_plain = timed(g_decode_plain, sub, 10)

    # ---- pack-once: once per round, then the steady
    # steps attend the dense packed cache instead of gathering the kept rows
    packed = [svl.pack_kv(Ks[l], Vs[l], seq, wl.vb, wl.nv, idxs[l]) for l in range(LAYERS)]
    ident = torch.arange(wl.k, dtype=torch.int32, device=dev).expand(wl.B, wl.Hkv, wl.k).contiguous()
    ws_p = svl.Workspace(dev)
    ws_p.get(1024)
    g_pack = graph_of(lambda: [svl.pack_kv(Ks[l], Vs[l], seq, wl.vb, wl.nv, idxs[l], Kp=packed[l][0],
                                           Vp=packed[l][1], ws=ws_p) for l in range(LAYERS)])
    g_decode_packed = graph_of(lambda: [svl.sparse_decode_attn(qds[l], packed[l][0], packed[l][1], packed[l][2],
                                                               wl.vb, wl.k, ident, out=outs[l], ws=ws_d,
                                                               flags=svl.SVL_DECODE_STATIC_PREFIX)
                                        for l in range(LAYERS)])
    ms_pack = timed(g_pack, sub, 10)
    ms_decode_packed = timed(g_decode_packed, sub, 10)
    T_att = wl.vb + wl.t_after
    pack_bytes = 2 * (2 * wl.B * wl.Hkv * (wl.k + T_att) * wl.d * 2)  # read + write of K and V rows
    del packed

    # ---- e2e through the public API with host buffers (pinned)
    qd_host = torch.stack(qds).cpu().pin_memory()
    newkv_host = torch.zeros(LAYERS, 2, wl.B, wl.Hkv, wl.d, dtype=torch.bfloat16).pin_memory()
    out_host = torch.empty(LAYERS, wl.B, wl.H, wl.d, dtype=torch.float32).pin_memory()
    qd_dev = torch.stack(qds)
    newkv_dev = torch.empty(LAYERS, 2, wl.B, wl.Hkv, wl.d, dtype=torch.bfloat16, device=dev)
    last = wl.seq_len - 1
    for l in range(LAYERS):
        newkv_host[l, 0] = Ks[l][:, :, last].cpu()
        newkv_host[l, 1] = Vs[l][:, :, last].cpu()
    qds_e = [qd_dev[l] for l in range(LAYERS)]

    kv_dst = [Ks[l][:, :, last] for l in range(LAYERS)] + [Vs[l][:, :, last] for l in range(LAYERS)]
    kv_src = [newkv_dev[l, 0] for l in range(LAYERS)] + [newkv_dev[l, 1] for l in range(LAYERS)]

    def e2e_step():
        # append the current token's K/V rows of every layer (one multi-tensor copy), then the
        # 28 fresh steps
        torch._foreach_copy_(kv_dst, kv_src)
        for l in range(LAYERS):
            svl.fresh_decode_step(qds_e[l], Ks[l], Vs[l], seq, wl.vb, wl.nv, wl.k,
                                  idx_out=idxs[l], out=outs[l], ws=ws_f)

    def e2e_step_io():
        # the same step with its host copies as graph nodes: pinned H2D of q and the new K/V
        # rows, the step, one D2H of the 28 layer outputs -- one replay per token
        qd_dev.copy_(qd_host, non_blocking=True)
        newkv_dev.copy_(newkv_host, non_blocking=True)
        e2e_step()
        out_host.copy_(out_all, non_blocking=True)

    try:
        g_e2e, e2e_in_graph = graph_of(e2e_step_io), True
    except RuntimeError:  # (copies not capturable here: issue them around the replay)
        torch.cuda.synchronize()
        g_e2e, e2e_in_graph = graph_of(e2e_step), False
    out_stack = torch.stack(outs)  # placeholder to size
    h2d = qd_host.numel() * 2 + newkv_host.numel() * 2
    d2h = out_host.numel() * 4
    e2e_steps = max(50, args.steps // 10)

    def e2e_once():
        if not e2e_in_graph:
            qd_dev.copy_(qd_host, non_blocking=True)
            newkv_dev.copy_(newkv_host, non_blocking=True)
        g_e2e.replay()
        if not e2e_in_graph:
            out_host.copy_(out_all, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    for _ in range(5):
        e2e_once()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_once()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
    _ = out_stack

    # ---- prefill companion (a6 salience, a7 per-frame prune) on the SURVEY.md 8(d) d2
    # "prune" config: 256 frames x 512 tokens, 16 encoder heads, d_e 72, s_p = 0.75
    prefill = None
    if rank == 0 and world == 1:
        pw = gen.PrefillWorkload()
        px = gen.make_prefill_inputs(pw, seed=7, device=dev)
        sal = torch.empty(pw.F, pw.Nf, dtype=torch.float32, device=dev)
        ws_p = svl.Workspace(dev)
        offs = [f * pw.Nf for f in range(pw.F + 1)]
        kept = torch.empty(1, svl.keep_budget(pw.Nf, pw.sparsity) * pw.F, dtype=torch.int32, device=dev)

        def sal_step():
            svl.salience(px["Qe"], px["Ke"], pw.S, svl.SVL_SAL_INTRA_VISUAL, out=sal, ws=ws_p)

        def prune_step():
            svl.prefill_prune(sal.view(1, -1), pw.sparsity, offs, kept_idx=kept, ws=ws_p)

        g_sal, g_prune = graph_of(sal_step), graph_of(prune_step)
        ms_sal = timed(g_sal, 20, 3)
        ms_prune = timed(g_prune, 200, 10)
        flops_exec = 2 * pw.Nf * pw.Nf * pw.de * pw.He * pw.F  # S = Q K^T once per head and frame (tcgen05)
        flops_survey = 2 * flops_exec  # SURVEY.md 8(d) d5 counts two QK^T passes
        bf16_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops") \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
        n_exp = pw.Nf * pw.Nf * pw.He * pw.F
        tf_exec = flops_exec / (ms_sal * 1e-3) / 1e12
        prefill = {"config": f"prune: {pw.F} frames x {pw.Nf} tokens, H_e {pw.He}, d_e {pw.de}, "
                             f"INTRA_VISUAL, s_p {pw.sparsity}",
                   "salience_ms": ms_sal,
                   "salience_tflops": tf_exec,
                   "salience_flops_accounting": "executed: 2 N_f^2 d_e per head and frame (the tcgen05 kernel "
                                                "computes S = Q K^T once; row LSE and column sums come from the "
                                                "same tile); SURVEY.md 8(d) d5's 2-pass count is "
                                                "salience_tflops_survey_count",
                   "salience_tflops_survey_count": flops_survey / (ms_sal * 1e-3) / 1e12,
                   "salience_exp2_per_s": n_exp / (ms_sal * 1e-3),
                   "salience_bound": "measured: exp2 + issue bound at d_e = 72 (one exponential per 2 d_e flop)",
                   "bf16_peak_tflops": bf16_peak,
                   "salience_frac": (tf_exec / bf16_peak) if bf16_peak else None,
                   "prune_us": ms_prune * 1e3, "kept": int(kept.numel())}
        # f4(i): unified RoPE remap of the kept tokens (pre-RoPE K rotated to their new
        # contiguous positions, V compacted) on the LLM cache the prune feeds: 4 KV heads, d 128
        rw = gen.CONFIGS[WORKLOAD]
        nvp, kp_ = int(pw.F * pw.Nf), int(kept.numel())
        capr = rw.vb + nvp + rw.t_after
        Kpre = torch.randn(1, rw.Hkv, capr, rw.d, device=dev).to(torch.bfloat16)
        Vpre = torch.randn(1, rw.Hkv, capr, rw.d, device=dev).to(torch.bfloat16)
        seqr = torch.tensor([capr], dtype=torch.int32, device=dev)
        kept_rel = kept.view(1, -1).contiguous()
        Kro, Vro, _ = svl.rope_remap(Kpre, Vpre, seqr, rw.vb, nvp, kept_rel, 1000000.0)
        g_rope = graph_of(lambda: svl.rope_remap(Kpre, Vpre, seqr, rw.vb, nvp, kept_rel, 1000000.0,
                                                 K_out=Kro, V_out=Vro, ws=ws_p))
        ms_rope = timed(g_rope, 50, 5)
        rope_bytes = 2 * 2 * rw.Hkv * (rw.vb + kp_ + rw.t_after) * rw.d * 2  # K, V rows read + written
        prefill.update({"rope_remap_us": ms_rope * 1e3, "rope_remap_GB_s": rope_bytes / (ms_rope * 1e-3) / 1e9,
                        "rope_remap_what": f"svl_rope_remap: {nvp} visual -> {kp_} kept + {rw.vb + rw.t_after} "
                                           f"text rows, {rw.Hkv} KV heads, d {rw.d}, base 1e6 (SURVEY 8(f) f4(i))"})
        # f4(i), multimodal RoPE: the same kept set on a 256-frame x 16 x 32 grid, Qwen2-VL sections
        tt, hh, ww = torch.meshgrid(torch.arange(pw.F), torch.arange(16), torch.arange(pw.Nf // 16), indexing="ij")
        coords = torch.stack([tt.reshape(-1), hh.reshape(-1), ww.reshape(-1)], -1).to(torch.int32).view(1, -1, 3).to(dev)
        ws_m = svl.Workspace(dev)
        Kmo, Vmo, _, _ = svl.mrope_remap(Kpre, Vpre, seqr, rw.vb, nvp, coords, kept_rel, 1000000.0, (16, 24, 24),
                                         ws=ws_m)
        g_mrope = graph_of(lambda: svl.mrope_remap(Kpre, Vpre, seqr, rw.vb, nvp, coords, kept_rel, 1000000.0,
                                                   (16, 24, 24), K_out=Kmo, V_out=Vmo, ws=ws_m))
        ms_mrope = timed(g_mrope, 50, 5)
        prefill.update({"mrope_remap_us": ms_mrope * 1e3, "mrope_remap_GB_s": rope_bytes / (ms_mrope * 1e-3) / 1e9,
                        "mrope_remap_what": "svl_mrope_remap: plan (per-dimension rank compression of the kept "
                                            "(t,h,w)) + sectioned re-rotation, 256 x 16 x 32 grid, sections "
                                            "(16, 24, 24) (SURVEY 8(f) f4(i), reading A23)"})
        del Kpre, Vpre, Kro, Vro, Kmo, Vmo

    # ---- question-chunk retrieval on tcgen05: svl_retrieve
    # with n_q question rows on the long-video cache, FULL_PREFIX normalisation computed in-kernel
    qret = None
    if rank == 0 and world == 1:
        base = gen.CONFIGS[WORKLOAD]
        bf16_peak_q = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops") \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
        runs = []
        for n_q in (32, 512):
            wq = gen.DecodeWorkload(**{**base.__dict__, "name": f"q{n_q}", "n_q": n_q, "seq_lens": None})
            xq = gen.make_decode_inputs(wq, seed=21, device=dev)
            ws_q = svl.Workspace(dev)
            idx_q = torch.empty(wq.B, wq.Hkv, wq.k, dtype=torch.int32, device=dev)

            def rq(xq=xq, wq=wq, ws_q=ws_q, idx_q=idx_q):
                svl.retrieve(xq["q"], xq["K"], xq["seq_len"], wq.vb, wq.nv, wq.k, idx_out=idx_q, ws=ws_q)

            ms_q = timed(graph_of(rq), 20, 3)
            # f1's attention output (svl_question_attention: row-LSE pass + output pass), alone and
            # followed by the retrieval on its LSE (lse_in: the column-mass pass reuses it)
            out_q = torch.empty(wq.B, n_q, wq.H, wq.d, dtype=torch.float32, device=dev)
            lse_q = torch.empty(wq.B, n_q, wq.H, dtype=torch.float32, device=dev)
            ws_a = svl.Workspace(dev)

            def ra(xq=xq, wq=wq, ws_a=ws_a, out_q=out_q, lse_q=lse_q):
                svl.question_attention(xq["q"], xq["K"], xq["V"], xq["seq_len"], wq.vb, wq.nv, out=out_q,
                                       lse_out=lse_q, ws=ws_a)

            def rar(xq=xq, wq=wq, ws_q=ws_q, idx_q=idx_q, lse_q=lse_q):
                ra()
                svl.retrieve(xq["q"], xq["K"], xq["seq_len"], wq.vb, wq.nv, wq.k, idx_out=idx_q, ws=ws_q,
                             lse_in=lse_q)

            ms_a = timed(graph_of(ra), 20, 3)
            ms_ar = timed(graph_of(rar), 20, 3)
            L, units = wq.seq_len, wq.B * wq.Hkv
            keys_p0 = wq.g * (n_q * (L - n_q) + n_q * (n_q + 1) // 2)  # causal prefix per query row
            flops_q = 2 * wq.d * units * (keys_p0 + n_q * wq.g * wq.nv)  # row-LSE pass + column-mass pass
            n_exp = units * (keys_p0 + 256 * ((n_q * wq.g + 255) // 256) * wq.nv)
            tf = flops_q / (ms_q * 1e-3) / 1e12
            flops_a = 6 * wq.d * units * keys_p0  # row-LSE pass (2d) + S and P.V of the output pass (4d)
            tf_a = flops_a / (ms_a * 1e-3) / 1e12
            runs.append({"n_q": n_q, "query_rows_per_unit": n_q * wq.g, "us": ms_q * 1e3, "tflops": tf,
                         "frac_bf16_peak": tf / bf16_peak_q if bf16_peak_q else None,
                         "exp2_per_s": n_exp / (ms_q * 1e-3),
                         "attention_output_us": ms_a * 1e3, "attention_output_tflops": tf_a,
                         "attention_output_frac_bf16_peak": tf_a / bf16_peak_q if bf16_peak_q else None,
                         "attention_then_retrieve_us": ms_ar * 1e3})
            del xq, ws_q, ws_a, out_q, lse_q
        qret = {"what": "svl_retrieve, n_q question rows (tensor-core path: row-LSE pass + column-mass pass + "
                        "cluster top-k), long-video cache (32768 visual + 768 text rows, 28/4 heads, d 128), "
                        "k = 3277 per KV group, one layer",
                "flops_accounting": "2 d per (query row, visible key) for each of the two passes; "
                                    "attention_output (svl_question_attention): 6 d per (query row, visible "
                                    "key) = row-LSE pass + S and P.V; attention_then_retrieve = the output "
                                    "call followed by svl_retrieve with its LSE as lse_in",
                "bound": "exp2 (SFU + FP32-pipe polynomial) at d = 128: one exponential per 256 flop",
                "bf16_peak_tflops": bf16_peak_q, "runs": runs}

    # ---- throughput sweep (BASELINE configs[4]: B = 16, 64k visual, k = 10 %): the fresh
    # step at 64k per unit runs the two-call path (score -> select -> decode); 3 rotating
    # layers of 1.3 GB each (> L2), single GPU
    sweep = None
    if rank == 0 and world == 1 and not args.profile:
        sw = gen.CONFIGS["sweep"]
        sxs = [gen.make_decode_inputs(sw, seed=900 + i, device=dev) for i in range(3)]
        ws_s = svl.Workspace(dev)
        ws_s.get(svl.fresh_decode_workspace_size(sw.B, sw.H, sw.Hkv, sw.d, sw.k, sw.nv, sw.capacity))
        sidx = torch.empty(sw.B, sw.Hkv, sw.k, dtype=torch.int32, device=dev)
        sout = torch.empty(sw.B, sw.H, sw.d, device=dev)
        g_sweep = graph_of(lambda: [svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], sw.vb, sw.nv,
                                                          sw.k, idx_out=sidx, out=sout, ws=ws_s) for x in sxs])
        ms_sw = timed(g_sweep, 20, 3) / len(sxs)
        sw_bytes = step_bytes(sw)["total"]
        sweep = {"config": "throughput sweep: B 16, 65536 visual, k 6554, 28/4 heads, d 128 (BASELINE configs[4])",
                 "us_per_layer": ms_sw * 1e3, "GB_s": sw_bytes / (ms_sw * 1e-3) / 1e9,
                 "hbm_frac_of_measured": sw_bytes / (ms_sw * 1e-3) / 1e9 / peaks()[0],
                 "bytes_per_layer": sw_bytes,
                 "path": "svl_fresh_decode_step -> two calls at 64k per unit (score, select, decode kernels)"}
        del sxs

    # ---- steady step (decode only, indices reused) and the per-round amortised step
    steady_us = ms_decode * 1e3 / LAYERS
    steady_bytes = nbytes["decode"]
    amort_us = (ms_step * 1e3 / LAYERS + (ROUND_STEPS - 1) * steady_us) / ROUND_STEPS
    pack_us, steady_packed_us = ms_pack * 1e3 / LAYERS, ms_decode_packed * 1e3 / LAYERS
    amort_packed_us = (ms_step * 1e3 / LAYERS + pack_us + (ROUND_STEPS - 1) * steady_packed_us) / ROUND_STEPS

    # ---- roofline of the dominant kernel (the fused fresh step)
    peak, peak_src = peaks()
    score_us = ms_score * 1e3 / LAYERS
    fused_us = ms_step * 1e3 / LAYERS
    achieved = nbytes["fused"] / (fused_us * 1e-6) / 1e9
    traffic, traffic_src = fresh_traffic()
    # ---- the other BASELINE configs as rows: nvila-4k and the multi-turn
    # round (8 rounds of 1 fresh retrieval + 249 steady steps, batch 8)
    rows = None
    pages = None
    if rank == 0 and world == 1 and not args.profile:
        rows = config_rows(graph_of, timed)
        pages = page_row(graph_of, timed)

    # ---- CPU baseline (rank 0, N=1 only): the oracle on all host cores, and on one thread
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, layers, th, secs = cpu_oracle_sample(wl)
        v1, layers1, _, secs1 = cpu_oracle_sample(wl, budget_s=4.0, nthreads=1)
        cpu = {"value": v / 1e9, "unit": "GB/s", "cores": th, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"{layers} whole layers of the long-video step (retrieve + sparse decode),"
                         f" {secs:.1f} s of fp64 oracle work, OpenMP over (b, KV-group) units",
               "one_thread": {"value": v1 / 1e9, "unit": "GB/s", "cores": 1,
                              "sample": f"{layers1} whole layers, {secs1:.1f} s"}}

    launches = LAYERS * args.steps  # one fused fresh_kernel launch per layer
    if rank == 0:
        line = {
            "metric": "decode step HBM GB/s (retrieve+sparse attn) @32k visual tok",
            "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded generator, paper_2510_17777_b200/inputs.py)",
            "config": config_dict(wl),
            "us_per_layer": ms_step * 1e3 / LAYERS,
            "ms_per_step_distribution": pct,
            "cold_single_layer_us": {"fresh_step": cold_fresh_us, "steady_decode": cold_decode_us,
                                     "how": "one launch after a 2 x L2 write, events around the launch only "
                                            "(no overlap with a neighbouring layer; SURVEY.md 8(d) d6)"},
            "tokens_per_s": wl.B * world / (ms_step * 1e-3),
            "hbm_frac_of_measured": value / world / peak,
            "unfused_us_per_layer": {"retrieve+decode (2 calls)": ms_unfused * 1e3 / LAYERS,
                                     "score": score_us, "select": ms_select * 1e3 / LAYERS,
                                     "decode+merge": ms_decode_plain * 1e3 / LAYERS},
            "bytes_per_layer": nbytes["total"],
            "steady": {"us_per_layer": steady_us, "GB_s": steady_bytes / (steady_us * 1e-6) / 1e9,
                       "bytes_per_layer": steady_bytes,
                       "what": "svl_sparse_decode_attn alone (selected + text K/V), indices reused, "
                               "SVL_DECODE_STATIC_PREFIX (rows below the current token's gathered before "
                               "the PDL wait, overlapping the previous layer's tail)",
                       "us_per_layer_without_early_gathers": ms_decode_plain * 1e3 / LAYERS},
            "amortized_us_per_layer": amort_us,
            "amortized_what": f"(1 fresh step + {ROUND_STEPS - 1} steady steps) / {ROUND_STEPS} per round",
            "pack_once": {"what": "svl_pack_kv once per round (kept visual + text K/V -> dense cache), then "
                                  "svl_sparse_decode_attn over the packed cache (SURVEY.md 8(f) f2)",
                          "pack_us_per_layer": pack_us,
                          "pack_GB_s": pack_bytes / (pack_us * 1e-6) / 1e9,
                          "steady_packed_us_per_layer": steady_packed_us,
                          "amortized_packed_us_per_layer": amort_packed_us},
            "roofline": {"bound": "hbm", "kernel": "fresh_kernel (svl_fresh_decode_step)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": nbytes["fused"]},
            "prefill": prefill,
            "question_retrieve": qret,
            "throughput_sweep": sweep,
            "configs": rows,
            "page_retrieval": pages,
            "cpu_baseline": cpu,
            "e2e": {"value": nbytes["total"] * LAYERS * world / (e2e_ms * 1e-3) / 1e9,
                    "unit": "GB/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "how": ("one CUDA-graph replay per token: " if e2e_in_graph else "")
                           + "pinned H2D of q + new K/V rows, the K/V appends (one multi-tensor copy) "
                           "+ 28 svl_fresh_decode_step calls, one D2H of the 28 layer outputs"
                           + (" (copies are graph nodes)" if e2e_in_graph else " (copies around the replay)")
                           + ", host wall clock"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
