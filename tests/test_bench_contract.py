"""bench.py's reference arm (runs on CPU: the oracle port on the host cores)
keeps the driver's JSON contract; a non-zero rank of a multi-rank launch
prints nothing and exits 0."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(extra_env=None):
    env = dict(os.environ, **(extra_env or {}))
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                           "--steps", "1", "--warmup", "0"], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=600)


def test_reference_arm_json_line():
    p = _run()
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]


def test_reference_arm_other_ranks_silent():
    p = _run({"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert p.returncode == 0, p.stderr[-2000:]
    assert not [l for l in p.stdout.splitlines() if l.startswith("{")]


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun launches two ranks itself (one per
    GPU; gloo plumbing run here) and rank 0 reports n_gpus = 2 with the
    max-over-ranks time -- the driver's scaling run cannot silently measure
    one GPU."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    assert d["ms_max_over_ranks"] >= 19.0  # rank 1 sleeps 20 ms: the max, not rank 0's


def test_gpus_flag_disagreeing_with_world_size_fails():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode == 2 and "disagrees" in p.stderr


def test_reference_arm_reports_host_info():
    d = json.loads([l for l in _run().stdout.splitlines() if l.startswith("{")][0])
    host = d["cpu_baseline"]["host"]
    assert host["cpu_count"] >= 1 and host["numpy"] and "threads_env" in host


def test_side_configs_record_failures(monkeypatch):
    """bench.side_configs embeds configs 3-5 from child processes; a child
    that fails, prints nothing or times out is recorded under its name instead
    of failing the config-2 line."""
    import importlib.util
    import subprocess as sp
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)

    calls = []

    def fake_run(cmd, capture_output, text, timeout):
        calls.append(cmd)
        name = cmd[cmd.index("--config") + 1] if "--config" in cmd else "cfg4"
        if name == "cfg3":
            return sp.CompletedProcess(cmd, 0, stdout='{"value": 4.0, "config": {"workload": "w3"}, '
                                                      '"p50_ttft_ms": 250.0, "extra": 1}\n', stderr="")
        if name == "cfg4":
            return sp.CompletedProcess(cmd, 1, stdout="", stderr="boom")
        raise sp.TimeoutExpired(cmd, timeout)

    monkeypatch.setattr(bench.subprocess, "run", fake_run)

    class A:
        side_timeout = 5
    out = bench.side_configs(A())
    assert len(calls) == 3
    assert out["cfg3"]["value"] == 4.0 and out["cfg3"]["workload"] == "w3"
    assert "extra" not in out["cfg3"] and out["cfg3"]["wall_s"] >= 0
    assert out["cfg4"]["error"].startswith("exit 1") and "boom" in out["cfg4"]["error"]
    assert "timed out" in out["cfg5"]["error"]
