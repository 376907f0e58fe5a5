#!/usr/bin/env python
"""Eager vs CUDA-graph replay of the selective-prefill engine: identical logits,
time per request for the HBM and pinned pools.  python tools/graph_check.py [LAYERS]"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_24022_b200 as ct  # noqa: E402
from paper_2605_24022_b200.pipeline import SelectivePrefillEngine  # noqa: E402
from paper_2605_24022_b200.pool import KvPool  # noqa: E402


def timeit(fn, n=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = ct.ModelConfig.llama3_8b(n_layers=L, seed=1234)
m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
rng = np.random.default_rng([0, 7])
chunks = [ct.encode_chunk_isolated(m, rng.integers(0, cfg.vocab_size, size=2048), chunk_id=f"c{j}")
          for j in range(16)]
ranks = ct.rank_chunks(chunks)
suffix_h = torch.as_tensor(rng.integers(0, cfg.vocab_size, size=64).astype(np.int32)).pin_memory()
suffix_d = suffix_h.cuda()
for loc in ("hbm", "pinned"):
    pool = KvPool(chunks, ranks, loc)
    eng = SelectivePrefillEngine(m, pool, 0.15, 64)
    out_h = torch.empty((1, cfg.vocab_size), dtype=torch.float32).pin_memory()
    src = suffix_h if loc == "pinned" else suffix_d
    eager = eng.step(src, out_h).clone()
    t_eager = timeit(lambda: eng.step(src, out_h))
    eng.capture(src, out_h)
    torch.cuda.synchronize()
    graph = eng.replay().clone()
    torch.cuda.synchronize()
    t_graph = timeit(lambda: eng.replay())
    print(f"{loc}: eager {t_eager:.2f} ms  graph {t_graph:.2f} ms  launches/step "
          f"{eng.launches_per_step}  identical={torch.equal(eager, graph)}  "
          f"host_copy_ok={torch.equal(out_h.cuda(), graph)}")
    del eng, pool
    torch.cuda.empty_cache()
