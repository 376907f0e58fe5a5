"""Selection-strategy experiment: attention recovery.

Mirrors ct/toymodel.py:344-419 on the device path: every strategy gets the
same recompute budget ceil(r*N) per chunk, the chunks are encoded in
isolation, the selective prefill runs through the CUDA kernels, and the
suffix rows' attention over the history is compared with a full recompute
(mean per-head Frobenius distance, ct/toymodel.py:113-124).

Strategies: "lowfreq" (the CacheTune scorer), "highfreq" (the complementary
band, device scorer with band=1), "random" (a seeded permutation — host
numpy draw identical to the reference's), "none" (reuse everything) and
"full" (recompute everything).  Models come from `GpuModel.reference_init`,
so a seed names the same ToyModel weights the reference draws.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from .errors import InvalidPlan
from .model import GpuModel, ModelConfig
from .prefill import attention_deviation, encode_chunk_isolated, full_prefill, selective_prefill
from .spectral import ImportanceRanking, rank_chunk

STRATEGIES = ("lowfreq", "highfreq", "random", "none", "full")


def strategy_ranking(chunk, strategy: str, alpha: float = 0.5,
                     rng: np.random.Generator | None = None) -> ImportanceRanking:
    """Token order a selection strategy recomputes first (ct/toymodel.py:351-371)."""
    if strategy in ("lowfreq", "none", "full"):
        return rank_chunk(chunk, alpha)
    if strategy == "highfreq":
        return rank_chunk(chunk, alpha, band="high")
    if strategy == "random":
        if rng is None:
            raise InvalidPlan("random strategy needs an rng")
        n = chunk.token_count
        perm = rng.permutation(n)
        scores = np.tile((n - np.argsort(perm)).astype(np.float64), (chunk.n_layers, 1))
        orders = np.tile(perm, (chunk.n_layers, 1))
        return ImportanceRanking(per_layer_scores=scores, per_layer_order=orders,
                                 aggregate_order=perm, alpha=alpha, n_tokens=n)
    raise InvalidPlan(f"unknown strategy {strategy!r}")


def effective_ratio(strategy: str, r: float) -> float:
    """ct/toymodel.py:374-379."""
    if strategy == "none":
        return 0.0
    if strategy == "full":
        return 1.0
    return r


def run_selection_experiment(seeds: Sequence[int], r: float = 0.15,
                             strategy: str = "lowfreq",
                             chunk_tokens: Sequence[int] = (64, 64, 64),
                             suffix_len: int = 8, alpha: float = 0.5, mlp: bool = False,
                             dtype=torch.float32) -> list[tuple[int, float]]:
    """Suffix-attention deviation from the full recompute, per seed
    (ct/toymodel.py:382-419; same seed-derived token ids and permutations)."""
    if strategy not in STRATEGIES:
        raise InvalidPlan(f"unknown strategy {strategy!r}")
    results = []
    for seed in seeds:
        cfg = ModelConfig(seed=seed, mlp=mlp)
        model = GpuModel.reference_init(cfg, dtype=dtype)
        tok_rng = np.random.default_rng([seed, 1])
        sel_rng = np.random.default_rng([seed, 2])
        chunk_ids = [tok_rng.integers(0, cfg.vocab_size, size=n) for n in chunk_tokens]
        suffix = tok_rng.integers(0, cfg.vocab_size, size=suffix_len)
        history = int(sum(chunk_tokens))
        full = full_prefill(model, np.concatenate(chunk_ids + [suffix]), record_attention=True)
        chunks = [encode_chunk_isolated(model, t, chunk_id=f"s{seed}-c{j}")
                  for j, t in enumerate(chunk_ids)]
        rankings = [strategy_ranking(c, strategy, alpha, rng=sel_rng) for c in chunks]
        sel = selective_prefill(model, chunks, rankings, suffix, effective_ratio(strategy, r),
                                record_attention=True)
        dev = attention_deviation(full.attention.suffix_view(history),
                                  sel.attention.suffix_view(history))
        results.append((seed, dev))
    return results
