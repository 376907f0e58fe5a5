#!/usr/bin/env python
"""Benchmark of the B200 selective-recompute prefill (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One step = one request of the configured workload (default config 2: Llama-3-8B
geometry, 16 chunks x 2048 tokens + 64-token suffix = 32K context, r = 0.15)
through the online path: selection plan -> QKV recompute of the selected rows
+ suffix -> deferred-RoPE blend of the reused KV -> tcgen05 attention ->
projections/MLP, 32 layers -> first-token logits.  Per rank, requests are
independent (replicas, weak scaling; no collective on the hot path).

value  = requests/s over all ranks, chunk pool resident in HBM.
e2e    = same metric with the pool in PINNED HOST memory: each step copies the
         keep rows (3.65 GB) host->HBM on the copy engines, the suffix tokens in
         and the logits out, all inside the timed region.
Timing: CUDA events on the launching stream, barrier + synchronize around the
timed region, max over ranks.  Inputs are larger than L2 (4.3 GB pool, 16 GB
weights), so no explicit L2 flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "p50 TTFT (ms) and prefill requests/sec at 32K ctx, 15% recompute; HBM GB/s & TC util"

CONFIGS = {
    "cfg2": dict(desc="config 2: Llama-3-8B geometry (32 layers, 32 q / 8 kv heads, D=128, "
                      "SwiGLU 14336, vocab 128256), 16 chunks x 2048 tokens + 64 suffix = "
                      "32832-token context, r=0.15, single B200",
                 arch="llama3_8b", layers=32, vocab=128256, chunks=16, chunk_tokens=2048,
                 suffix=64, r=0.15),
    "cfg3": dict(desc="config 3: Mistral-7B geometry, 32 chunks x 2048 tokens + 64 suffix = "
                      "65600-token context, r=0.15",
                 arch="mistral_7b", layers=32, vocab=32768, chunks=32, chunk_tokens=2048,
                 suffix=64, r=0.15),
    "cfg5": dict(desc="config 5: batch of 64 independent RAG requests, each 16 chunks x 2048 "
                      "tokens drawn from a shared 64-chunk importance-ordered KV corpus resident "
                      "in HBM (Llama-3-8B geometry) + its own 64-token suffix, r=0.15; request i "
                      "-> rank i mod N (strong scaling: the batch is fixed)",
                 arch="llama3_8b", layers=32, vocab=128256, chunks=16, chunk_tokens=2048,
                 suffix=64, r=0.15, corpus=64, requests=64),
    "small": dict(desc="reduced smoke workload: Llama-3-8B layer geometry, 2 layers, "
                       "4 chunks x 2048 + 64", arch="llama3_8b", layers=2, vocab=8192,
                  chunks=4, chunk_tokens=2048, suffix=64, r=0.15),
}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"],
                    bf16_sust=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sust=1400.0, src="fallback (B200_PROFILING.md)")


def ncu_traffic(kernel: str, config: str):
    """DRAM bytes per launch from the committed ncu capture (profiles/ncu_traffic.json);
    only meaningful for the config the capture was taken on (config 2)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if config != "cfg2" or not p.exists():
        return None
    entry = json.loads(p.read_text()).get(kernel)
    return None if entry is None else entry["bytes"]


def ncu_field(kernel: str, field: str, config: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if config != "cfg2" or not p.exists():
        return None
    entry = json.loads(p.read_text()).get(kernel) or {}
    v = entry.get(field)
    return None if v is None else v / 100.0


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return False
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)
        return False

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------- CPU arm

def cpu_sample(cfgname: str, seed: int = 0, rows: int = 256):
    """Bounded sample of the reference CPU path (oracle port, float64 numpy):
    one layer of config `cfgname` for `rows` active query rows (uniformly spread
    over the request's real positions) + that layer's full deferred-RoPE fuse,
    extrapolated linearly to all active rows and all layers.  Returns
    (seconds_per_request_extrapolated, description)."""
    from oracle import cachetune_oracle as O
    c = CONFIGS[cfgname]
    hq, hkv, d, inter = 32, 8, 128, 14336
    hid = hq * d
    N, C, S = c["chunk_tokens"], c["chunks"], c["suffix"]
    k = O.selection_count(c["r"], N)
    n_ctx = C * N + S
    A = C * k + S
    rng = np.random.default_rng(seed)
    sc = 1.0 / np.sqrt(hid)
    W = {n: rng.uniform(-1, 1, size=s) * sc for n, s in
         (("wq", (hid, hid)), ("wk", (hid, hkv * d)), ("wv", (hid, hkv * d)),
          ("wo", (hid, hid)), ("wg", (hid, inter)), ("wu", (hid, inter)), ("wd", (inter, hid)))}
    pos = np.sort(rng.choice(C * N, size=C * k, replace=False))
    pos = np.concatenate([pos, np.arange(C * N, n_ctx)])
    sample_pos = pos[np.linspace(0, A - 1, rows).astype(int)]
    h = rng.standard_normal((rows, hid))
    k_raw = rng.standard_normal((n_ctx - A, hkv, d)).astype(np.float32)
    v_keep = rng.standard_normal((n_ctx - A, hkv, d)).astype(np.float32)
    keep = np.setdiff1d(np.arange(n_ctx), pos)
    rope = O.Rope(d)
    t0 = time.perf_counter()
    # fuse: deferred RoPE of every reused row + scatter with the recomputed rows
    x = O.rms_norm(h)
    q = (x @ W["wq"]).reshape(rows, hq, d)
    kk = (x @ W["wk"]).reshape(rows, hkv, d)
    vv = (x @ W["wv"]).reshape(rows, hkv, d)
    q_rot = O.rope_rotate(q, sample_pos, rope)
    k_rot = O.rope_rotate(kk, sample_pos, rope)
    t_lin0 = time.perf_counter() - t0
    t1 = time.perf_counter()
    kbuf = np.zeros((n_ctx, hkv, d), np.float32)
    vbuf = np.zeros((n_ctx, hkv, d), np.float32)
    kbuf[keep] = O.rope_apply(k_raw, keep, rope)
    vbuf[keep] = v_keep
    t_fuse = time.perf_counter() - t1
    t2 = time.perf_counter()
    kc, vc = kbuf.astype(np.float64), vbuf.astype(np.float64)
    causal = np.arange(n_ctx)[None, :] <= sample_pos[:, None]
    ctx, _ = O._attention(q_rot, kc, vc, causal, hq, hkv, d, False)
    h = h + ctx.reshape(rows, hid) @ W["wo"]
    xm = O.rms_norm(h)
    g = xm @ W["wg"]
    h = h + ((g / (1 + np.exp(-g))) * (xm @ W["wu"])) @ W["wd"]
    t_rest = time.perf_counter() - t2
    per_layer = t_fuse + (t_lin0 + t_rest) * (A / rows)
    del k_rot, vv
    desc = (f"oracle port (float64 numpy/OpenBLAS) on one layer of {cfgname}: {rows} of {A} "
            f"active rows (uniform over positions) + the layer's full fuse of {n_ctx - A} reused "
            f"rows; extrapolated x{A / rows:.0f} rows x{c['layers']} layers")
    return per_layer * c["layers"], desc, t_fuse + t_lin0 + t_rest


def cfg1_end_to_end(repeats: int = 3) -> dict:
    """Config 1 end to end on both sides: the 2-layer
    toy model, 4 chunks x 512 tokens + 32 suffix, r = 0.15.  CPU = the oracle
    port of the reference (rank_chunk x 4 + selective_prefill, float64 numpy,
    the reference runs this config as-is); GPU = the drop-in API on host
    inputs (rank_chunk x 4 + selective_prefill, fp32 mode, H2D/D2H included).
    Best of `repeats`; the GPU logits are checked against the oracle's."""
    import torch
    import paper_2605_24022_b200 as ct
    from oracle import cachetune_oracle as O
    om = O.Model(O.ModelConfig(seed=0, n_layers=2))
    rng = np.random.default_rng([0, 1])
    toks = [rng.integers(0, 256, size=512) for _ in range(4)]
    suffix = rng.integers(0, 256, size=32)
    ochunks, chunks = [], []
    for j, t in enumerate(toks):
        kr, vs = O.encode_chunk_isolated(om, t)
        ochunks.append((kr, vs, t))
        chunks.append(ct.KvChunk(f"c{j}", tuple(ct.SeqTensor(k) for k in kr),
                                 tuple(ct.SeqTensor(v) for v in vs), source_tokens=t))
    gm = ct.GpuModel.from_reference(om, dtype=torch.float32)

    # the reference's own semantics on both sides: PrefillResult with the
    # attention record and the logits of every active row (ct/toymodel.py:223-311)
    def cpu_once():
        aggs = [O.rank_chunk(kr, vs)[2] for kr, vs, _ in ochunks]
        return O.selective_prefill(om, ochunks, aggs, suffix, 0.15)

    def gpu_once():
        ranks = [ct.rank_chunk(c) for c in chunks]
        res = ct.selective_prefill(gm, chunks, ranks, suffix, 0.15).to_host()
        return res.logits

    gpu_once()
    torch.cuda.synchronize()
    t_gpu, t_cpu = [], []
    for _ in range(repeats):
        t0 = time.perf_counter()
        got = gpu_once()
        t_gpu.append(time.perf_counter() - t0)
    with all_host_threads():
        for _ in range(repeats):
            t0 = time.perf_counter()
            want = cpu_once()
            t_cpu.append(time.perf_counter() - t0)
    err = O.normwise_rel(np.asarray(got, np.float64), want["logits"])
    return {"workload": "config 1: 2-layer toy model (H=2, D=8), 4 chunks x 512 + 32 suffix, "
                        "r = 0.15, rank_chunk x 4 + selective_prefill end to end",
            "gpu_ms": min(t_gpu) * 1e3, "cpu_ms": min(t_cpu) * 1e3,
            "cpu_kind": "port", "cpu_cores": cpu_threads(),
            "speedup": min(t_cpu) / min(t_gpu), "logits_normwise_err": err,
            "note": "wall clock, best of %d; both sides return the attention record and every "
                    "active row's logits; GPU = drop-in API on host KvChunks (fp32 mode, copies "
                    "included), a launch-bound toy shape" % repeats}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def all_host_threads():
    """BLAS thread pool sized to every host core this process may use (torchrun
    exports OMP_NUM_THREADS=1, which numpy's OpenBLAS would otherwise honour)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=cpu_threads())
    except ImportError:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()


def host_info() -> dict:
    """CPU model, core counts, numpy / BLAS versions and the thread environment
    the CPU arm ran with."""
    info = {"cpu_count": os.cpu_count(), "affinity": cpu_threads(),
            "threads_env": {k: os.environ.get(k) for k in
                            ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}}
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    info["numpy"] = np.__version__
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads")}
                        for d in threadpool_info() if d.get("user_api") == "blas"]
    except ImportError:  # pragma: no cover
        pass
    return info


def pinned_h2d_peak(dev) -> float:
    """GB/s of one 1 GiB contiguous pinned-host -> HBM copy (best of 3)."""
    import torch
    src = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    best = float("inf")
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dst.copy_(src, non_blocking=True)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    del src, dst
    return (1 << 30) / (best * 1e-3) / 1e9


def run_reference(args, rank, world):
    """The reference's CPU path (oracle port) on the host cores.  A step is
    one bounded sample (cpu_sample): `ms_per_step` is its measured wall time,
    `value` the requests/s it extrapolates to (the sample covers
    `request_fraction_per_step` of a request's work)."""
    c = CONFIGS[args.config]
    if rank != 0:
        return
    req_s, step_s = [], []
    desc = ""
    with all_host_threads():
        for i in range(args.warmup + args.steps):
            r, desc, st = cpu_sample(args.config, seed=i, rows=args.cpu_rows)
            if i >= args.warmup:
                req_s.append(r)
                step_s.append(st)
    sec = statistics.median(req_s)
    step = statistics.median(step_s)
    val = 1.0 / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "requests/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step * 1000.0, "request_fraction_per_step": step / sec,
        "p50_ttft_ms_extrapolated": sec * 1000.0, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": c["desc"]}, "sample": desc,
        "cpu_baseline": {"value": val, "unit": "requests/s", "cores": cpu_threads(),
                         "kind": "port", "sample": desc, "host": host_info()},
        "e2e": {"value": val, "unit": "requests/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm

def run_ours(args, rank, world, local_rank):
    from paper_2605_24022_b200.distributed import bind_to_gpu_numa
    import torch
    import torch.distributed as dist
    import paper_2605_24022_b200 as ct
    from paper_2605_24022_b200 import _lib
    from paper_2605_24022_b200.pipeline import (FullPrefillEngine, KernelTimer,
                                                SelectivePrefillEngine)
    from paper_2605_24022_b200.offline import encode_and_rank, encode_batch
    from paper_2605_24022_b200.pool import KvPool
    from paper_2605_24022_b200.spectral import score_device, score_select_fast, selection_count

    c = CONFIGS[args.config]
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    # N > 1: each rank on its GPU's NUMA node before the pinned pool is touched
    numa_cpus = bind_to_gpu_numa(dev.index) if world > 1 else None
    peaks = load_peaks()
    log = (lambda *a: print(*a, file=sys.stderr, flush=True)) if rank == 0 else (lambda *a: None)

    arch = getattr(ct.ModelConfig, c["arch"])
    cfg = arch(n_layers=c["layers"], vocab_size=c["vocab"], seed=1234)
    t0 = time.time()
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16, device=dev)
    # independent requests per rank (weak scaling): rank-seeded token streams
    rng = np.random.default_rng([rank, 7])
    toks = [rng.integers(0, cfg.vocab_size, size=c["chunk_tokens"]) for _ in range(c["chunks"])]
    suffix = rng.integers(0, cfg.vocab_size, size=c["suffix"]).astype(np.int32)
    # offline stage: encode straight into the scorer's
    # [C, L, N, Hkv, D] batch, score it, one permute launch builds the pool
    ids = [f"r{rank}c{j}" for j in range(len(toks))]
    keys, vals, chunks = encode_batch(model, toks, ids)  # warm-up + the batch buffers
    torch.cuda.synchronize()
    e_enc = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e_enc[0].record()
    encode_batch(model, toks, ids, out=(keys, vals))
    e_enc[1].record()
    torch.cuda.synchronize()
    encode_ms = e_enc[0].elapsed_time(e_enc[1])
    # the same with each chunk's exact scorer overlapped on a side stream
    # (the scorer is FP-pipe bound, the encode tensor-pipe bound)
    encode_and_rank(model, toks[:1], 0.5, "f64", ids[:1])  # warm-up of the side-stream path
    torch.cuda.synchronize()
    e_ov = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e_ov[0].record()
    ov = encode_and_rank(model, toks, 0.5, "f64", ids, out=(keys, vals))
    e_ov[1].record()
    torch.cuda.synchronize()
    encode_rank_ms = e_ov[0].elapsed_time(e_ov[1])
    ov_agg = ov[3]["agg_order"]
    del ov
    log(f"[bench] model + {len(chunks)} encoded chunks in {time.time() - t0:.1f}s")

    # (1) scorer (offline stage): f64 exact mode over the request's chunks
    sc_times = {}
    k_sel = selection_count(c["r"], c["chunk_tokens"])
    scorers = {"f64": lambda: score_device(keys, vals, 0.5, "f64", want_layer_order=False),
               "fast": lambda: score_select_fast(keys, vals, k_sel)}
    for prec, fn in scorers.items():
        for _ in range(2):  # warm-up (first launches load the kernels)
            fn()
        ms_list = []
        for _ in range(5):  # median of individually timed calls
            torch.cuda.synchronize()
            es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            es.record()
            out = fn()
            ee.record()
            torch.cuda.synchronize()
            ms_list.append(es.elapsed_time(ee))
        sc_times[prec] = statistics.median(ms_list)
        if prec == "f64":
            agg_rows = out["agg_order"]
        else:  # the certified top-k sets must be the exact ones
            fast_wcount = out["wcount"].cpu().numpy()
            fast_exact = bool(torch.equal(
                torch.sort(out["agg_order"][:, :k_sel], dim=1).values,
                torch.sort(agg_rows[:, :k_sel], dim=1).values))
    rankings = []
    for j, ch in enumerate(chunks):
        # device aggregate order feeds the pool; host arrays only for the drop-in type
        n = ch.token_count
        rankings.append(ct.ImportanceRanking(
            per_layer_scores=np.zeros((1, n)), per_layer_order=np.arange(n)[None, :],
            aggregate_order=agg_rows[j].cpu().numpy().astype(np.int64), alpha=0.5,
            n_tokens=n, device_aggregate=agg_rows[j]))
    scorer_bytes = keys.numel() * keys.element_size() * 2

    KvPool(chunks[:1], rankings[:1], "hbm", device=dev)  # warm-up
    pool_hbm = KvPool(chunks, rankings, "hbm", device=dev)
    permute_ms = pool_hbm.permute_ms  # device time of the one permute launch
    permute_bytes = 2 * scorer_bytes  # every K/V byte read once and written once
    nch = len(chunks)
    offline = {
        "chunks": nch, "chunk_tokens": c["chunk_tokens"],
        "encode_ms_per_chunk": encode_ms / nch,
        "score_f64_ms_per_chunk": None, "score_fast_ms_per_chunk": None,
        "encode_rank_overlapped_ms_per_chunk": encode_rank_ms / nch,
        "permute_ms_per_chunk": permute_ms / nch,
        "permute_launches": pool_hbm.permute_launches,
        "permute": {"bound": "hbm", "bytes": permute_bytes,
                    "achieved": permute_bytes / (permute_ms * 1e-3) / 1e9,
                    "peak": peaks["hbm"], "unit": "GB/s",
                    "frac": permute_bytes / (permute_ms * 1e-3) / 1e9 / peaks["hbm"]},
        "overlapped_orders_equal": bool(torch.equal(ov_agg, agg_rows)),
        "note": "encode writes K/V into the [C, L, N, Hkv, D] scorer batch; one scorer launch "
                "set; one ct_pool_permute launch writes the importance-ordered pool.  "
                "encode_rank_overlapped = encode with each chunk's exact (f64) scorer on a side "
                "stream behind it (offline.encode_and_rank)",
    }
    del keys, vals
    pool_pin = KvPool(chunks, rankings, "pinned", device=dev,
                      resident_layers=args.resident_layers)
    del chunks
    torch.cuda.empty_cache()
    timer = KernelTimer()
    eng = SelectivePrefillEngine(model, pool_hbm, c["r"], c["suffix"], timer=timer)
    eng_e2e = SelectivePrefillEngine(model, pool_pin, c["r"], c["suffix"])
    suffix_dev = torch.as_tensor(suffix, device=dev)
    suffix_host = torch.as_tensor(suffix).pin_memory()
    logits_host = torch.empty((1, cfg.vocab_size), dtype=torch.float32).pin_memory()
    log(f"[bench] pools ready (A={eng.A}, n_ctx={eng.n_ctx}, keep/chunk={eng.n_keep}) "
        f"{time.time() - t0:.1f}s")

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(fn, steps):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record()
        for s, e in evs:
            s.record()
            fn()
            e.record()
        g1.record()
        torch.cuda.synchronize()
        barrier()
        return [s.elapsed_time(e) for s, e in evs], g0.elapsed_time(g1)

    for _ in range(args.warmup):
        eng.step(suffix_dev)
        eng_e2e.step(suffix_host, logits_host)
    torch.cuda.synchronize()
    log(f"[bench] warmup done {time.time() - t0:.1f}s")

    # ---- value: pool resident in HBM
    timer.enabled = True
    launches0 = _lib.LAUNCH_COUNT["n"]
    with ClockSampler(local_rank) as clk:
        step_ms, total_ms = timed(lambda: eng.step(suffix_dev), args.steps)
    launches = (_lib.LAUNCH_COUNT["n"] - launches0)
    timer.enabled = False
    att_ms = timer.mean_ms("attention")
    blend_ms = timer.mean_ms("blend")
    qkv_ms = timer.mean_ms("qkv")
    mlp_ms = timer.mean_ms("mlp_gemm")  # nan when the fused MLP does not run
    qkvg_ms = timer.mean_ms("qkv_gemm")  # nan when the fused QKV GEMM does not run
    # ---- e2e: pinned host pool, H2D keep rows + tokens, D2H logits, all timed
    e2e_ms, e2e_total = timed(lambda: eng_e2e.step(suffix_host, logits_host), args.steps)
    # ---- the same requests replayed from CUDA graphs (the engines' public
    # capture() / replay(): one graph launch per request instead of ~300 host
    # launches; H2D of the keep rows and suffix, D2H of the logits still run
    # inside every replay).  These are the headline value / e2e when enabled;
    # the eager numbers above stay in the line under "eager" and carry the
    # per-kernel events.
    g = None
    if not args.no_graph:
        eng.capture(suffix_dev)
        eng_e2e.capture(suffix_host, logits_host)
        for _ in range(args.warmup):
            eng.replay()
            eng_e2e.replay()
        launches_g0 = _lib.LAUNCH_COUNT["n"]
        with ClockSampler(local_rank) as clk_g:
            g_step_ms, g_total_ms = timed(lambda: eng.replay(), args.steps)
        g = {"launches": _lib.LAUNCH_COUNT["n"] - launches_g0, "clk": clk_g}
        g_e2e_ms, g_e2e_total = timed(lambda: eng_e2e.replay(), args.steps)
        eager = {"ms_per_step": total_ms / args.steps, "p50_ttft_ms": statistics.median(step_ms),
                 "e2e_p50_ttft_ms": statistics.median(e2e_ms), "gpu_launches": launches,
                 "clocks": clk.summary()}
        step_ms, total_ms, e2e_ms, e2e_total = g_step_ms, g_total_ms, g_e2e_ms, g_e2e_total
        launches, clk = g["launches"], g["clk"]
    # sparse transfer alone (copy engines, after the timed regions): one
    # request's streamed keep tails, and a plain contiguous pinned H2D copy as
    # the measured peak
    h2d_ms = statistics.median(eng_e2e.time_transfer() for _ in range(3))
    h2d_peak = pinned_h2d_peak(dev)
    ref_logits = eng.step(suffix_dev).float()
    torch.cuda.synchronize()
    agree = float((logits_host.to(dev) - ref_logits).abs().max() /
                  ref_logits.abs().max().clamp_min(1e-30))
    # ---- full-recompute baseline, same kernels
    full_ms = None
    e2e_h2d = eng_e2e.h2d_bytes
    eng_ring = eng_e2e.ring
    stage_bytes = eng_e2e.stage.numel() * eng_e2e.stage.element_size()
    copies_per_req = (cfg.n_layers - eng_e2e.res) * eng_e2e.C
    if not args.no_full:
        del eng_e2e
        torch.cuda.empty_cache()
        full = FullPrefillEngine(model, eng.n_ctx)
        all_tok = torch.cat([pool_hbm.tokens.reshape(-1), suffix_dev]).contiguous()
        full.step(all_tok)
        fms, _ = timed(lambda: full.step(all_tok), max(1, min(2, args.steps)))
        full_ms = statistics.median(fms)
        del full
        torch.cuda.empty_cache()

    # ---- result gather off the hot path (config 5: first-token logits,
    # selected positions, TTFT of every rank's request to rank 0 over NCCL)
    from paper_2605_24022_b200.distributed import RequestResult, gather_results
    g0 = time.perf_counter()
    gathered = gather_results(
        [RequestResult(rank, statistics.median(step_ms), ref_logits[0].float(),
                       eng.positions[:eng.n_rec].clone())], cfg.vocab_size, eng.n_rec, device=dev)
    gather_ms = (time.perf_counter() - g0) * 1e3

    # ---- aggregate over ranks (max of times)
    def allmax(x):
        if world == 1 or x is None:
            return x
        t = torch.tensor([float(x)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    total_ms = allmax(total_ms)
    e2e_total = allmax(e2e_total)
    if g is not None:
        for k in ("ms_per_step", "p50_ttft_ms", "e2e_p50_ttft_ms"):
            eager[k] = allmax(eager[k])
        eager["value"] = world * 1e3 / eager["ms_per_step"]
    p50 = allmax(statistics.median(step_ms))
    p50_e2e = allmax(statistics.median(e2e_ms))
    full_ms = allmax(full_ms)
    h2d_ms = allmax(h2d_ms)
    att_ms = allmax(att_ms)
    blend_ms = allmax(blend_ms)
    qkv_ms = allmax(qkv_ms)
    mlp_ms = allmax(mlp_ms)
    qkvg_ms = allmax(qkvg_ms)
    sc64 = allmax(sc_times["f64"])
    scfast = allmax(sc_times["fast"])
    if rank != 0:
        return
    offline["score_f64_ms_per_chunk"] = sc64 / nch
    offline["score_fast_ms_per_chunk"] = scfast / nch

    L = cfg.n_layers
    att_flops = eng.attention_flops_per_layer()
    att_tflops = att_flops / (att_ms * 1e-3) / 1e12
    mlp_flops = 2.0 * eng.A * cfg.hidden_dim * 2 * cfg.inter
    # x read + W_gu read + act written (bf16)
    mlp_floor = 2 * (eng.A * cfg.hidden_dim + cfg.hidden_dim * 2 * cfg.inter + eng.A * cfg.inter)
    blend_bytes = eng.blend_bytes_per_layer()
    blend_gbs = blend_bytes / (blend_ms * 1e-3) / 1e9
    # QKV epilogue: read q|k|v rows, write q + cache K + cache V (+ no raw K here)
    qkv_bytes = 2 * eng.A * (cfg.n_heads + 2 * cfg.kv_heads) * cfg.head_dim * 2
    qkv_gbs = qkv_bytes / (qkv_ms * 1e-3) / 1e9
    qkvg_flops = 2.0 * eng.A * cfg.hidden_dim * (cfg.n_heads + 2 * cfg.kv_heads) * cfg.head_dim
    # scorer: exact mode is FP64-pipe bound.  Algorithmic work = a forward and
    # an inverse complex FFT (split-radix 4N log2 N - 6N + 8 flops) per packed
    # pair of lanes; peak = 64 DFMA lanes/clk/SM x 2 x 148 SMs x max SM clock.
    n_tok = c["chunk_tokens"]
    n_sig = c["chunks"] * cfg.n_layers * 2 * (cfg.kv_heads * cfg.head_dim // 2)
    sc_flops = n_sig * 2 * (4 * n_tok * np.log2(n_tok) - 6 * n_tok + 8)
    fp64_peak = 64 * 2 * 148 * 1.965e9 / 1e12
    value = world * args.steps / (total_ms * 1e-3)
    e2e_val = world * args.steps / (e2e_total * 1e-3)
    # FLOPs actually performed per request: every layer projects q|k|v for all
    # A rows (the last layer's K/V complete the blended cache), but the last
    # layer's attention / O-projection / MLP run on the final row only -- the
    # first-token logits read nothing else (prefill.run_layers, prune_last);
    # the full-recompute baseline is pruned the same way.
    def request_flops(rows, att_per_layer, last_pos):
        qkv_w = sum(layer["wqkv"].numel() for layer in model.layers)
        rest_w = sum(w.numel() for layer in model.layers for k, w in layer.items() if k != "wqkv")
        rest_last = sum(w.numel() for k, w in model.layers[-1].items() if k != "wqkv")
        return (2.0 * rows * qkv_w + 2.0 * rows * (rest_w - rest_last) + 2.0 * rest_last
                + 2.0 * cfg.hidden_dim * cfg.vocab_size + att_per_layer * (L - 1)
                + 4.0 * cfg.n_heads * cfg.head_dim * (last_pos + 1))
    step_flops = request_flops(eng.A, att_flops, eng.n_ctx - 1)
    full_flops = None
    if full_ms is not None:
        n = eng.n_ctx
        full_flops = request_flops(n, 4.0 * cfg.n_heads * cfg.head_dim * n * (n + 1) / 2, n - 1)

    cpu = None
    if world == 1 and not args.no_cpu:
        with all_host_threads():
            sec, desc, _ = cpu_sample(args.config, rows=args.cpu_rows)
        cpu = {"value": 1.0 / sec, "unit": "requests/s", "cores": cpu_threads(), "kind": "port",
               "sample": desc, "host": host_info()}
        try:
            cpu["cfg1_end_to_end"] = cfg1_end_to_end()
        except Exception as e:  # reported, never silently dropped
            cpu["cfg1_end_to_end"] = {"error": f"{type(e).__name__}: {e}"}
    line = {
        "metric": METRIC, "value": value, "unit": "requests/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "p50_ttft_ms": p50, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights, seeded token ids; chunk KV "
                                 "encoded on the GPU by the same model)",
        "config": {"workload": c["desc"], "parallelism": f"replicas x{world} (request-level)",
                   "numa_bind": (f"{len(numa_cpus)} GPU-local cpus" if numa_cpus else None),
                   "pool": "importance-ordered, HBM-resident (value) / pinned host (e2e)",
                   "l2": "inputs larger than L2 (4.3 GB pool + 16 GB weights); no flush",
                   "active_rows": eng.A, "n_ctx": eng.n_ctx, "keep_rows_per_chunk": eng.n_keep},
        "roofline": {"kernel": "ct_selective_attention (tcgen05)", "bound": "tensor",
                     "achieved": att_tflops, "peak": peaks["bf16_sust"], "unit": "TFLOP/s",
                     "frac": att_tflops / peaks["bf16_sust"],
                     "traffic": ncu_traffic("attention_pp_kernel", args.config),
                     "flops_per_launch": att_flops, "launch_ms": att_ms,
                     "peak_source": peaks["src"] + " bf16 sustained",
                     # per-clock utilisation from the committed ncu capture:
                     # at D = 128 the tensor and MUFU work per key block are
                     # equal (profiles/round2_attention_probes.md)
                     "tensor_pipe_active_ncu": ncu_field("attention_pp_kernel",
                                                         "tensor_pipe_pct", args.config),
                     "mufu_pipe_active_ncu": ncu_field("attention_pp_kernel",
                                                       "mufu_pipe_pct", args.config)},
        "kernels": {
            "gather_rope_blend": {"bound": "hbm", "achieved": blend_gbs, "peak": peaks["hbm"],
                                  "unit": "GB/s", "frac": blend_gbs / peaks["hbm"],
                                  "bytes_per_launch": blend_bytes, "launch_ms": blend_ms,
                                  "traffic": ncu_traffic("blend_bf16_kernel", args.config)},
            # separate QKV epilogue kernel: only when the fused QKV GEMM is off
            "qkv_rope_scatter": (None if not np.isfinite(qkv_ms) else {
                "bound": "hbm", "achieved": qkv_gbs, "peak": peaks["hbm"],
                "unit": "GB/s", "frac": qkv_gbs / peaks["hbm"],
                "bytes_per_launch": qkv_bytes, "launch_ms": qkv_ms,
                "traffic": ncu_traffic("qkv_bf16_kernel", args.config)}),
            # q|k|v GEMM with RoPE + cache scatter in the epilogue
            # (ct_gemm_qkv_rope): 2 A hid (Hq + 2 Hkv) D flops per launch
            "qkv_gemm_rope": (None if not np.isfinite(qkvg_ms) else {
                "bound": "tensor", "achieved": qkvg_flops / (qkvg_ms * 1e-3) / 1e12,
                "peak": peaks["bf16_sust"], "unit": "TFLOP/s",
                "frac": qkvg_flops / (qkvg_ms * 1e-3) / 1e12 / peaks["bf16_sust"],
                "flops_per_launch": qkvg_flops, "launch_ms": qkvg_ms,
                "traffic": ncu_traffic("gemm_qkv_rope_kernel", args.config)}),
            # MLP gate/up GEMM + SwiGLU epilogue (ct_gemm_swiglu, tcgen05 CTA
            # pairs): 2 A hid 2I flops per launch, timed per launch in-step
            "mlp_gate_up_swiglu": (None if not np.isfinite(mlp_ms) else {
                "bound": "tensor", "achieved": mlp_flops / (mlp_ms * 1e-3) / 1e12,
                "peak": peaks["bf16_sust"], "unit": "TFLOP/s",
                "frac": mlp_flops / (mlp_ms * 1e-3) / 1e12 / peaks["bf16_sust"],
                "flops_per_launch": mlp_flops, "launch_ms": mlp_ms,
                "hbm_floor_bytes": mlp_floor,
                "traffic": ncu_traffic("gemm_swiglu_kernel", args.config)}),
            "scorer_f64_per_request": {
                "ms": sc64, "bytes": scorer_bytes, "bound": "fp64 (exact mode)",
                "hbm_gbs": scorer_bytes / (sc64 * 1e-3) / 1e9,
                "hbm_frac": scorer_bytes / (sc64 * 1e-3) / 1e9 / peaks["hbm"],
                "algorithmic_gflop": sc_flops / 1e9,
                "achieved_tflops": sc_flops / (sc64 * 1e-3) / 1e12,
                "fp64_peak_tflops": fp64_peak,
                "fp64_frac": sc_flops / (sc64 * 1e-3) / 1e12 / fp64_peak,
                "fp64_pipe_busy_ncu": ncu_field("fft2_energy_kernel_f64", "fp64_pipe_pct",
                                                args.config),
                "note": "exact (f64) mode is FP64-pipe bound: achieved/peak counts split-radix "
                        "flops (a DADD is 1 flop), the pipe-busy figure is from the committed "
                        "ncu capture",
                "traffic": ncu_traffic("fft2_energy_kernel_f64", args.config)},
            "scorer_fast_per_request": {
                "ms": scfast, "bytes": scorer_bytes, "bound": "fp32 pipe (ops/B above the ridge)",
                "hbm_gbs": scorer_bytes / (scfast * 1e-3) / 1e9,
                "hbm_frac": scorer_bytes / (scfast * 1e-3) / 1e9 / peaks["hbm"],
                "fp32_pipe_busy_ncu": ncu_field("fs_energy_split_kernel", "fma_pipe_pct", args.config),
                "selection_equals_exact": fast_exact,
                "chunks_certified_by_guard": int((fast_wcount == 0).sum()),
                "chunks_rescored": int((fast_wcount > 0).sum()),
                "chunks_exact_fallback": int((fast_wcount < 0).sum()),
                "note": "single-precision four-step FFT scores + certified top-k boundary "
                        "(window tokens re-scored in float64); orders exact at k",
                "traffic": ncu_traffic("fs_energy_split_kernel", args.config)},
        },
        "offline": offline,
        "step_tflops": step_flops / (p50 * 1e-3) / 1e12,
        "sparse_h2d": {
            "bound": "pcie", "bytes_per_request": e2e_h2d, "copy_engine_ms": h2d_ms,
            "achieved": e2e_h2d / (h2d_ms * 1e-3) / 1e9 if h2d_ms else None,
            "peak": h2d_peak, "unit": "GB/s",
            "frac": (e2e_h2d / (h2d_ms * 1e-3) / 1e9 / h2d_peak) if h2d_ms else None,
            "peak_source": "measured here: one 1 GiB pinned->device cudaMemcpyAsync, best of 3",
            "exposed_ms": p50_e2e - p50,
            "ring_slots": eng_ring, "stage_bytes": stage_bytes,
            "resident_layers": args.resident_layers,
            "copies_per_request": copies_per_req,
            "note": "one cudaMemcpyAsync per (chunk, streamed layer) on a copy stream; exposed "
                    "= e2e p50 - HBM-pool p50 (the transfer time not hidden by compute)"},
        "e2e": {"value": e2e_val, "unit": "requests/s", "p50_ttft_ms": p50_e2e,
                "h2d_bytes_per_step": e2e_h2d + 4 * c["suffix"],
                "d2h_bytes_per_step": 4 * cfg.vocab_size, "logits_match_hbm_path": agree},
        "full_recompute_ttft_ms": full_ms,
        "ttft_speedup_vs_full": (full_ms / p50) if full_ms else None,
        "flop_ratio_bound": (full_flops / step_flops) if full_flops else None,
        "gpu_launches": launches,
        "timing": ("CUDA-graph replay of each request (SelectivePrefillEngine.capture/replay)"
                   if g is not None else "eager launches"),
        "eager": eager if g is not None else None,
        "result_gather": {"requests": len(gathered) if gathered else 0, "ms": gather_ms,
                          "note": "all_gather of logits/selections/TTFT after the timed region"},
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    return line


def run_batch(args, rank, world, local_rank):
    """Config 5: one step = the whole batch of independent requests, sharded
    i -> rank i mod N with no collective on the hot path.  Every rank holds a
    replica of the model and of the shared chunk corpus (its importance-ordered
    KV pool in HBM); a request binds its 16 documents and runs the online path.
    value = batch requests / max-over-ranks step time; e2e = the same with each
    request's suffix tokens and chunk ids from pinned host memory and its
    first-token logits back to pinned host memory inside the timed region."""
    import torch
    import torch.distributed as dist
    import paper_2605_24022_b200 as ct
    from paper_2605_24022_b200 import _lib
    from paper_2605_24022_b200.distributed import (RequestResult, bind_to_gpu_numa,
                                                   gather_results, shard_requests)
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool

    c = CONFIGS[args.config]
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    # N > 1: each rank on its GPU's NUMA node before the pinned pool is touched
    numa_cpus = bind_to_gpu_numa(dev.index) if world > 1 else None
    log = (lambda *a: print(*a, file=sys.stderr, flush=True)) if rank == 0 else (lambda *a: None)
    arch = getattr(ct.ModelConfig, c["arch"])
    cfg = arch(n_layers=c["layers"], vocab_size=c["vocab"], seed=1234)
    t0 = time.time()
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16, device=dev)
    corpus = []
    for j in range(c["corpus"]):  # same corpus on every rank (document seeds)
        toks = np.random.default_rng([j, 5]).integers(0, cfg.vocab_size, size=c["chunk_tokens"])
        corpus.append(ct.encode_chunk_isolated(model, toks, chunk_id=f"doc{j}"))
    ranks = ct.rank_chunks(corpus)
    pool = KvPool(corpus, ranks, "hbm", device=dev)
    del corpus
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    log(f"[bench] corpus of {c['corpus']} chunks encoded, ranked, pooled {time.time() - t0:.1f}s")
    mine = shard_requests(c["requests"], rank, world)
    reqs = {}
    for i in mine:
        rng = np.random.default_rng([i, 11])
        docs = [int(x) for x in rng.choice(c["corpus"], size=c["chunks"], replace=False)]
        suf = rng.integers(0, cfg.vocab_size, size=c["suffix"]).astype(np.int32)
        reqs[i] = (docs, torch.as_tensor(suf, device=dev), torch.as_tensor(suf).pin_memory())
    # CT_CFG5_STREAMS=k: k engines on k streams, requests dealt round-robin, so
    # one request's HBM-bound kernels can overlap another's tensor-core work
    n_streams = max(1, int(os.environ.get("CT_CFG5_STREAMS", "1")))
    engines = [SelectivePrefillEngine(model, pool, c["r"], c["suffix"], n_chunks=c["chunks"])
               for _ in range(n_streams)]
    eng = engines[0]
    streams = [torch.cuda.current_stream(dev)] if n_streams == 1 else \
        [torch.cuda.Stream(device=dev) for _ in range(n_streams)]
    logits_host = {i: torch.empty((1, cfg.vocab_size), dtype=torch.float32).pin_memory()
                   for i in mine}

    def batch(e2e=False, out=None):
        main = torch.cuda.current_stream(dev)
        for st in streams:
            st.wait_stream(main)
        for idx, i in enumerate(mine):
            docs, sd, sh = reqs[i]
            e = engines[idx % n_streams]
            with torch.cuda.stream(streams[idx % n_streams]):
                e.bind(docs)
                if e2e:
                    e.step(sh, logits_host[i])
                else:
                    lg = e.step(sd)
                    if out is not None:
                        out[i] = lg
        for st in streams:
            main.wait_stream(st)
    for _ in range(args.warmup):
        batch()
    torch.cuda.synchronize()

    def timed(fn):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            fn()
        e.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return s.elapsed_time(e)

    req_ms = []
    launches0 = _lib.LAUNCH_COUNT["n"]
    with ClockSampler(local_rank) as clk:
        total = timed(batch)
    launches = _lib.LAUNCH_COUNT["n"] - launches0
    e2e_total = timed(lambda: batch(e2e=True))
    # per-request TTFT (after the timed regions)
    last = {}
    for i in mine:
        docs, sd, _ = reqs[i]
        eng.bind(docs)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        last[i] = eng.step(sd)
        e.record()
        torch.cuda.synchronize()
        req_ms.append(s.elapsed_time(e))
    g0 = time.perf_counter()
    gathered = gather_results([RequestResult(i, req_ms[j], last[i][0].float(),
                                             eng.positions[:eng.n_rec].clone())
                               for j, i in enumerate(mine)], cfg.vocab_size, eng.n_rec, device=dev)
    gather_ms = (time.perf_counter() - g0) * 1e3

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([float(x)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    total, e2e_total = allmax(total), allmax(e2e_total)
    p50 = allmax(statistics.median(req_ms))
    if rank != 0:
        return
    n_req = c["requests"]
    cpu = None
    if world == 1 and not args.no_cpu:
        with all_host_threads():
            sec, desc, _ = cpu_sample(args.config, rows=args.cpu_rows)
        cpu = {"value": 1.0 / sec, "unit": "requests/s", "cores": cpu_threads(), "kind": "port",
               "sample": desc, "host": host_info()}
    line = {
        "metric": METRIC, "value": n_req * args.steps / (total * 1e-3), "unit": "requests/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / args.steps, "p50_ttft_ms": p50, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, seeded document and suffix token ids; corpus KV "
                "encoded on the GPU by the same model)",
        "config": {"workload": c["desc"], "parallelism": f"replicas x{world} (request-level)",
                   "numa_bind": (f"{len(numa_cpus)} GPU-local cpus" if numa_cpus else None),
                   "requests_per_step": n_req, "requests_on_rank0": len(mine), "streams": n_streams,
                   "l2": "inputs larger than L2 (17 GB corpus + 16 GB weights); no flush"},
        "e2e": {"value": n_req * args.steps / (e2e_total * 1e-3), "unit": "requests/s",
                "h2d_bytes_per_step": n_req * 4 * (c["suffix"] + c["chunks"]),
                "d2h_bytes_per_step": n_req * 4 * cfg.vocab_size},
        "gpu_launches": launches,
        "result_gather": {"requests": len(gathered) if gathered else 0, "ms": gather_ms},
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


SIDE_KEEP = ("value", "unit", "p50_ttft_ms", "ms_per_step", "steps", "warmup", "e2e",
             "roofline", "sparse_h2d", "full_recompute_ttft_ms", "ttft_speedup_vs_full",
             "flop_ratio_bound", "gpu_launches", "clocks", "scaling", "n_gpus")


def side_configs(args) -> dict:
    """Configs 3, 4 and 5 measured in the same (default, N = 1) run, each in
    its own process after the config-2 timed region, so the driver's record
    carries them: config 3 (64K context, pinned pool), config 4 (ratio sweep +
    the tuner over real GPU TTFTs, tools/ratio_sweep.py) and config 5 (the
    64-request batch).  A failure is recorded, it does not fail the line."""
    me = str(Path(__file__).resolve())
    jobs = {
        "cfg3": [me, "--config", "cfg3", "--steps", "3", "--warmup", "3", "--no-cpu",
                 "--side-configs", "none"],
        "cfg4": [str(ROOT / "tools" / "ratio_sweep.py"), "--steps", "3"],
        "cfg5": [me, "--config", "cfg5", "--steps", "2", "--warmup", "3", "--no-cpu",
                 "--side-configs", "none"],
    }
    out = {}
    for name, cmd in jobs.items():
        t0 = time.time()
        try:
            res = subprocess.run([sys.executable, *cmd], capture_output=True, text=True,
                                 timeout=args.side_timeout)
            rows = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
            if res.returncode != 0 or not rows:
                out[name] = {"error": f"exit {res.returncode}: {res.stderr.strip()[-300:]}"}
                continue
            d = json.loads(rows[-1])
            if name != "cfg4":
                d = {"workload": d.get("config", {}).get("workload"),
                     **{k: d[k] for k in SIDE_KEEP if k in d}}
            d["wall_s"] = round(time.time() - t0, 1)
            out[name] = d
        except subprocess.TimeoutExpired:
            out[name] = {"error": f"timed out after {args.side_timeout} s"}
        print(f"[bench] side config {name}: {time.time() - t0:.0f}s", file=sys.stderr,
              flush=True)
    return out


def self_launch(n: int) -> int:
    """Re-exec this script under torch.distributed.run with n ranks on this
    node (rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator sizes in the log (nranks check)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def run_dry(args, rank, world):
    """The launch / reduction plumbing of run_ours without the workload."""
    import torch
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo")
    t0 = time.perf_counter()
    time.sleep(0.01 * (rank + 1))
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world,
                          "ms_max_over_ranks": float(ms[0]), "steps": args.steps,
                          "warmup": args.warmup}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-full", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches only (no CUDA-graph replay)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=256)
    ap.add_argument("--resident-layers", type=int, default=0,
                    help="e2e arm: first n layers of the pinned pool also kept in HBM")
    ap.add_argument("--side-configs", default="auto", choices=["auto", "none"],
                    help="auto: a default config-2 run on one GPU also measures configs 3, "
                         "4 and 5 (separate processes, after the timed region) and embeds "
                         "them under 'configs'")
    ap.add_argument("--side-timeout", type=int, default=420)
    ap.add_argument("--dry-run", action="store_true",
                    help="plumbing only: rank/world handling and the max-over-ranks line, "
                         "no GPU work (CPU test of the multi-rank launch)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        # `bench.py --gpus N` outside torchrun: launch the N ranks ourselves
        # (one process per GPU) instead of silently measuring one GPU
        sys.exit(self_launch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} disagrees with WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, max(world, args.gpus))
        return
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # CT_BENCH_DIST=gloo + ranks folded onto the visible GPUs: a functional
        # check of the multi-rank path on a one-GPU box (its timings mean nothing)
        backend = os.environ.get("CT_BENCH_DIST", "nccl")
        # communicator sizes in the log (the driver's nranks check), also when
        # the driver launches the ranks with torchrun itself
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        if backend != "nccl":
            local_rank %= torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        if "requests" in CONFIGS[args.config]:
            run_batch(args, rank, world, local_rank)
        else:
            line = run_ours(args, rank, world, local_rank)
            if line is not None:
                if (args.side_configs == "auto" and args.config == "cfg2" and world == 1):
                    import gc
                    import torch
                    gc.collect()
                    torch.cuda.empty_cache()  # the config-2 model and pools are released
                    line["configs"] = side_configs(args)
                print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
