"""Tuner (scheduler) and pipeline simulator against traces produced by the live
reference (tests/golden/scheduler_cases.npz).  CPU only."""

import math

import numpy as np
import pytest

from conftest import golden
from paper_2605_24022_b200 import pipesim as P
from paper_2605_24022_b200 import scheduler as S
from paper_2605_24022_b200.errors import InvalidParam, ObjectiveError, ProfileError


def _cases():
    g = golden("scheduler_cases")
    return g, int(g["count"])


def test_gss_trace_matches_reference():
    g, n = _cases()
    for i in range(n):
        t_c, t_i, t_o = g[f"g{i}_p"]
        p = S.HardwareProfile(float(t_c), float(t_i), float(t_o))
        r_min, r_max, eps = g[f"g{i}_cfg"]
        cfg = S.SearchConfig(float(r_min), float(r_max), float(eps))
        r0 = S.roofline_r0(p, cfg)
        assert r0 == float(g[f"g{i}_r0"])
        r_star, evals, trace = S.gss_optimize(lambda r: S.ttft_model(r, 1000, 8, p), r0, cfg)
        assert r_star == float(g[f"g{i}_rstar"])
        assert np.array_equal(np.array(trace), g[f"g{i}_trace"])
        assert evals <= S.gss_eval_budget(cfg)


def test_simulate_matches_reference():
    g, n = _cases()
    for i in range(n):
        p = S.HardwareProfile(*map(float, g[f"g{i}_p"]))
        plan = P.synthetic_plan([100, 37, 64], 6, float(g[f"g{i}_sim_ratio"]), 2, 8)
        tl = P.simulate(plan, p)
        assert np.array_equal(np.array([[e.start_s, e.end_s] for e in tl.events]), g[f"g{i}_sim"])
        assert tl.ttft_s == float(g[f"g{i}_sim_ttft"])
        assert P.validate_timeline(tl, plan) == []
        assert tl.ttft_s <= P.serialized_ttft(plan, p) + 1e-15
        bw, lat = g[f"g{i}_tier"]
        tier = next(t for t in P.TIER_PRESETS.values() if t.read_bw == bw and t.fixed_latency == lat)
        tl2 = P.simulate(plan, p, tier=tier)
        assert np.array_equal(np.array([[e.start_s, e.end_s] for e in tl2.events]),
                              g[f"g{i}_sim_tier"])


def test_calibrate_with_sim_evaluator_matches_reference():
    g, n = _cases()
    for i in range(n):
        p = S.HardwareProfile(*map(float, g[f"g{i}_p"]))
        r_min, r_max, eps = g[f"g{i}_cfg"]
        cfg = S.SearchConfig(float(r_min), float(r_max), float(eps))
        bw, lat = g[f"g{i}_tier"]
        tier = next(t for t in P.TIER_PRESETS.values() if t.read_bw == bw and t.fixed_latency == lat)
        ev = P.make_sim_evaluator(p, tier=tier)
        cal = [P.RequestSpec(chunk_tokens=(128, 128, 128), n_layers=4)] * 3
        rep = S.calibrate(None, None, ev, cal, cfg, profile=p)
        assert rep.r_star == float(g[f"g{i}_cal_rstar"])
        assert np.array_equal(np.array(rep.trace), g[f"g{i}_cal_trace"])
        assert "r_star=" in rep.to_text()


def test_known_answers_and_validation():
    # tests/test_scheduler.py worked examples: 2150 us and 40 ms
    p = S.HardwareProfile(t_c=2e-6, t_i=1e-6, t_o=150e-6)
    assert math.isclose(S.per_layer_latency(0.5, 2000, p), 2150e-6)
    assert math.isclose(S.ttft_model(0.0, 1000, 8, S.HardwareProfile(1e-6, 5e-6)), 40e-3)
    with pytest.raises(InvalidParam):
        S.HardwareProfile(0.0, 1.0)
    with pytest.raises(InvalidParam):
        S.SearchConfig(r_min=0.5, r_max=0.4)
    with pytest.raises(ObjectiveError):
        S.gss_optimize(lambda r: float("nan"), 0.5, S.SearchConfig())
    with pytest.raises(InvalidParam):
        S.gss_optimize(lambda r: r, 0.95, S.SearchConfig())
    with pytest.raises(ProfileError):
        S.calibrate(None, None, lambda s, r: r, [1], S.SearchConfig())


def test_gss_matches_grid_on_random_profiles():
    rng = np.random.default_rng(404)
    cfg = S.SearchConfig()
    grid = np.arange(cfg.r_min, cfg.r_max + 1e-12, 0.001)
    for _ in range(100):
        p = S.HardwareProfile(float(rng.uniform(0.1e-6, 100e-6)), float(rng.uniform(0.1e-6, 100e-6)),
                              float(rng.uniform(0, 1e-3)))
        vals = 8 * np.maximum(grid * 1000 * p.t_c, (1 - grid) * 1000 * p.t_i) + 8 * p.t_o
        best = grid[int(np.argmin(vals))]
        r_star, evals, _ = S.gss_optimize(lambda r: S.ttft_model(r, 1000, 8, p),
                                          S.roofline_r0(p, cfg), cfg)
        assert evals <= 12 and abs(r_star - best) <= cfg.epsilon + 1e-3


def test_transferred_bytes_example():
    # tests/test_pipesim.py:73-79: 3264-byte transfer arithmetic
    plan = P.synthetic_plan([20, 31], 2, 0.15, n_heads=2, head_dim=4)
    keep = (20 - 3) + (31 - 5)
    assert P.transferred_bytes(plan) == keep * 2 * 4 * 4 * 2 * 2


def test_timeline_csv_round_trip():
    plan = P.synthetic_plan([64, 64], 4, 0.3)
    tl = P.simulate(plan, S.HardwareProfile(1e-6, 2e-6, 1e-5))
    csv = P.timeline_to_csv(tl)
    assert csv.splitlines()[0] == "stream,layer,start_s,end_s,label"
    assert len(csv.splitlines()) == 1 + 3 * 4


def test_transfer_cost_matches_reference_model(tmp_path):
    """Pool transfer profiling (ct/cachepool.py:489-529): analytic tiers give
    read_time / tokens exactly; a file-backed tier times a real read (> 0)."""
    from paper_2605_24022_b200.errors import InvalidParam
    from paper_2605_24022_b200.pipesim import TIER_PRESETS, TierConfig
    from paper_2605_24022_b200.pool import transfer_cost_per_token
    bpt = 8 * 128 * 4 * 2
    for name, tier in TIER_PRESETS.items():
        got = transfer_cost_per_token(tier, 1 << 20, bpt)
        assert got == tier.read_time(1 << 20) / ((1 << 20) / bpt), name
    disk = TierConfig("ssd", read_bw=535e6, write_bw=445e6, backing=str(tmp_path))
    assert transfer_cost_per_token(disk, 1 << 18, bpt) > 0
    assert not (tmp_path / ".transfer_probe").exists()
    import pytest
    with pytest.raises(InvalidParam):
        transfer_cost_per_token(disk, 0, bpt)


def test_tier_config_files_round_trip(tmp_path):
    """save/load_tier_config + resolve_tier (ct/cachepool.py:100-145)."""
    from paper_2605_24022_b200.errors import InvalidParam
    from paper_2605_24022_b200.pipesim import (TIER_PRESETS, TierConfig, load_tier_config,
                                               resolve_tier, save_tier_config)
    tier = TierConfig("ssd", read_bw=535e6, write_bw=445e6, fixed_latency=2e-4,
                      backing=str(tmp_path / "pool"))
    path = tmp_path / "tier.cfg"
    save_tier_config(tier, path)
    assert path.read_text().splitlines() == [
        "kind=ssd", "read_bw_bytes=535000000", "write_bw_bytes=445000000",
        "fixed_latency_s=0.0002", f"backing={tmp_path / 'pool'}"]
    assert load_tier_config(path) == tier
    assert resolve_tier(str(path)) == tier
    assert resolve_tier("hdd") == TIER_PRESETS["hdd"]
    (tmp_path / "bad.cfg").write_text("# c\nkind=ssd\nread_bw_bytes 5\n")
    import pytest
    with pytest.raises(InvalidParam):
        load_tier_config(tmp_path / "bad.cfg")
    (tmp_path / "short.cfg").write_text("kind=ssd\n")
    with pytest.raises(InvalidParam):
        load_tier_config(tmp_path / "short.cfg")
    with pytest.raises(InvalidParam):
        resolve_tier("nvram")
