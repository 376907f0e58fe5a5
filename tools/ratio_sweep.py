#!/usr/bin/env python
"""BASELINE config 4: recompute-ratio sweep 5%-50% at 32K context on one B200,
with the adaptive tuner picking the ratio from the B200-measured cost model.

For each r: p50 TTFT with the pool in HBM and in pinned host memory (sparse
PCIe transfer overlapped with recompute).  Then `profile_b200` fits
(t_c, t_i, t_o), `calibrate` runs the golden-section search over REAL measured
TTFTs (make_gpu_evaluator, pinned pool) with SearchConfig(r_min=.05,
r_max=.5, eps=.01), and the simulator's prediction is printed beside it.
Prints one JSON object.
"""

import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_24022_b200 as ct  # noqa: E402
from paper_2605_24022_b200 import pipesim, scheduler  # noqa: E402
from paper_2605_24022_b200.pipeline import SelectivePrefillEngine  # noqa: E402
from paper_2605_24022_b200.pool import KvPool  # noqa: E402


def p50_ttft(eng, steps=3):
    eng.step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        eng.step()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--chunks", type=int, default=16)
    ap.add_argument("--steps", type=int, default=3, help="timed steps per ratio (p50)")
    args = ap.parse_args()
    cfg = ct.ModelConfig.llama3_8b(n_layers=args.layers, seed=1234)
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng([0, 7])
    toks = [rng.integers(0, cfg.vocab_size, size=2048) for _ in range(args.chunks)]
    chunks = [ct.encode_chunk_isolated(model, t, chunk_id=f"c{j}") for j, t in enumerate(toks)]
    ranks = ct.rank_chunks(chunks)
    pool_hbm = KvPool(chunks, ranks, "hbm")
    pool_pin = KvPool(chunks, ranks, "pinned")
    del chunks
    torch.cuda.empty_cache()
    sweep = []
    for r in [0.05, 0.10, 0.15, 0.20, 0.25, 0.30, 0.35, 0.40, 0.45, 0.50]:
        row = {"r": r}
        for name, pool in (("hbm", pool_hbm), ("pinned", pool_pin)):
            eng = SelectivePrefillEngine(model, pool, r, 64)
            row[f"ttft_ms_{name}"] = p50_ttft(eng, args.steps)
            del eng
            torch.cuda.empty_cache()
        sweep.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    prof = scheduler.profile_b200(model, pool_pin)
    n = pool_pin.C * pool_pin.N
    scfg = scheduler.SearchConfig(r_min=0.05, r_max=0.5, epsilon=0.01)
    ev = scheduler.make_gpu_evaluator(model, pool_pin)
    rep = scheduler.calibrate(None, None, ev, ["request-0"], scfg, profile=prof)
    sim = pipesim.make_sim_evaluator(prof)
    spec = pipesim.RequestSpec(tuple([pool_pin.N] * pool_pin.C), pool_pin.L, pool_pin.H,
                               pool_pin.D)
    best = min(sweep, key=lambda x: x["ttft_ms_pinned"])
    out = {
        "workload": f"config 4: Llama-3-8B geometry, {args.chunks}x2048 + 64, ratio sweep",
        "sweep": sweep,
        "profile_b200": {"t_c_s": prof.t_c, "t_i_s": prof.t_i, "t_o_s": prof.t_o,
                         "h2d_gbs": 2 * pool_pin.row_bytes / prof.t_i / 1e9},
        "roofline_r0": scheduler.roofline_r0(prof, scfg),
        "calibrated_r_star": rep.r_star, "eval_count": rep.eval_count,
        "calibration_trace": rep.trace,
        "sim_ttft_ms_at_r_star": 1e3 * sim(spec, rep.r_star),
        "model_ttft_ms_at_r_star": 1e3 * scheduler.ttft_model(rep.r_star, n, pool_pin.L, prof),
        "grid_best_r_pinned": best["r"],
        "calibration_wall_s": rep.wall_time_s,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
