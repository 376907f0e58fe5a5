#!/usr/bin/env python
"""One profiled request of the bench workload, for ncu.

    ncu --profile-from-start off ... python tools/profile_step.py [--what step|scorer|full]

Builds the config-2 engine exactly like bench.py, runs one warm-up request,
then brackets ONE request (or one scorer pass / full prefill) with
cudaProfilerStart/Stop so ncu sees only that launch list.
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2605_24022_b200 as ct  # noqa: E402
from paper_2605_24022_b200.pipeline import FullPrefillEngine, SelectivePrefillEngine  # noqa: E402
from paper_2605_24022_b200.pool import KvPool  # noqa: E402
from paper_2605_24022_b200.spectral import score_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="step",
                    choices=["step", "scorer", "scorer32", "full", "busy"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--chunks", type=int, default=16)
    args = ap.parse_args()
    cfg = ct.ModelConfig.llama3_8b(n_layers=args.layers, seed=1234)
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng([0, 7])
    toks = [rng.integers(0, cfg.vocab_size, size=2048) for _ in range(args.chunks)]
    suffix = torch.as_tensor(rng.integers(0, cfg.vocab_size, size=64).astype(np.int32),
                             device="cuda")
    chunks = [ct.encode_chunk_isolated(model, t, chunk_id=f"c{j}") for j, t in enumerate(toks)]
    keys = torch.stack([c.keys for c in chunks])
    vals = torch.stack([c.values for c in chunks])
    if args.what.startswith("scorer"):
        prec = "f32" if args.what == "scorer32" else "f64"
        score_device(keys, vals, 0.5, prec, want_layer_order=False)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        score_device(keys, vals, 0.5, prec, want_layer_order=False)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    ranks = ct.rank_chunks(chunks)
    del keys, vals
    if args.what == "full":
        full = FullPrefillEngine(model, args.chunks * 2048 + 64)
        tok = torch.cat([torch.cat([c.tokens for c in chunks]), suffix])
        full.step(tok)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        full.step(tok)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    pool = KvPool(chunks, ranks, "hbm")
    del chunks
    eng = SelectivePrefillEngine(model, pool, 0.15, 64)
    eng.step(suffix)
    torch.cuda.synchronize()
    if args.what == "busy":
        busy(eng, suffix)
        return
    torch.cuda.profiler.start()
    eng.step(suffix)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


def busy(eng, suffix, steps: int = 3):
    """GPU busy fraction of back-to-back requests at full concurrency (CUPTI
    kernel + memcpy intervals via torch.profiler, not serialised like ncu):
    the union of device intervals vs the span from the first start to the
    last end, and the largest idle gaps with the activity that follows."""
    from torch.profiler import ProfilerActivity, profile
    for _ in range(2):
        eng.step(suffix)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            eng.step(suffix)
        torch.cuda.synchronize()
    ev = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                 if e.device_type.name == "CUDA"), key=lambda x: x[0])
    if not ev:
        print("no device activity recorded")
        return
    t0, t1 = ev[0][0], max(e[1] for e in ev)
    busy_us, cur_s, cur_e, gaps = 0.0, ev[0][0], ev[0][1], []
    for s, e, n in ev[1:]:
        if s > cur_e:
            busy_us += cur_e - cur_s
            gaps.append((s - cur_e, n))
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    busy_us += cur_e - cur_s
    span = t1 - t0
    print(f"{steps} requests: span {span / 1e3:.3f} ms, device busy {busy_us / 1e3:.3f} ms "
          f"({100 * busy_us / span:.1f} %), idle {(span - busy_us) / 1e3:.3f} ms in "
          f"{len(gaps)} gaps")
    for g, n in sorted(gaps, reverse=True)[:15]:
        print(f"  gap {g:9.1f} us before {n[:90]}")


if __name__ == "__main__":
    main()
