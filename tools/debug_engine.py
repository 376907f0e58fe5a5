#!/usr/bin/env python
"""Run a few selective-prefill requests of a given geometry with checks on.

    CUDA_LAUNCH_BLOCKING=1 python tools/debug_engine.py LAYERS CHUNKS R hbm|pinned [VOCAB] [STEPS]
"""
import sys
import traceback
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_24022_b200 as ct  # noqa: E402
from paper_2605_24022_b200.pipeline import SelectivePrefillEngine  # noqa: E402
from paper_2605_24022_b200.pool import KvPool  # noqa: E402

L, C, r, loc = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), sys.argv[4]
V = int(sys.argv[5]) if len(sys.argv) > 5 else 8192
steps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
cfg = ct.ModelConfig.llama3_8b(n_layers=L, vocab_size=V, seed=1)
m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
rng = np.random.default_rng(0)
chunks = [ct.encode_chunk_isolated(m, rng.integers(0, V, size=2048), chunk_id=f"c{j}")
          for j in range(C)]
ranks = ct.rank_chunks(chunks)
pool = KvPool(chunks, ranks, loc)
del chunks
eng = SelectivePrefillEngine(m, pool, r, 64)
suffix = torch.as_tensor(rng.integers(0, V, size=64).astype(np.int32)).pin_memory()
out = torch.empty((1, V), dtype=torch.float32).pin_memory()
try:
    for i in range(steps):
        eng.step(suffix, out)
        torch.cuda.synchronize()
        print("step", i, "ok", float(out.abs().max()))
    print("ok", L, C, r, loc, eng.A, eng.n_ctx)
except Exception:
    traceback.print_exc()
