"""fp32 mode (the 1e-5 tolerance mode) at full config-2 context: Llama-3-8B
layer geometry, 2 layers, 16 x 2048 chunks + 64 suffix = 32,832 tokens,
r = 0.15.  Both layers' blended caches vs the float64 oracle fuse_layer and
64 sampled attention rows x 8 q heads vs the float64 oracle attention:
max|d| / max|ref| <= 1e-5."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

C, N, S, R = 16, 2048, 64, 0.15


def test_fp32_mode_fullsize_context_vs_oracle():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2605_24022_b200 as ct
    from fullsize_oracle import check_request
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    cfg = ct.ModelConfig.llama3_8b(n_layers=2, vocab_size=4096, seed=21)
    m = ct.GpuModel.random(cfg, dtype=torch.float32)
    rng = np.random.default_rng(21)
    toks = [rng.integers(0, cfg.vocab_size, size=N) for _ in range(C)]
    chunks = [ct.encode_chunk_isolated(m, t, chunk_id=f"f{j}") for j, t in enumerate(toks)]
    ranks = ct.rank_chunks(chunks)
    suffix = torch.as_tensor(rng.integers(0, cfg.vocab_size, size=S).astype(np.int32),
                             device="cuda")
    eng = SelectivePrefillEngine(m, KvPool(chunks, ranks, "hbm"), R, S)
    errs = check_request(eng, chunks, suffix, (0, 1), seed=5, tol_attn=1e-5, tol_blend=1e-5)
    print("fp32 cfg2-context oracle errors", errs)
