"""bench.py's reference arm on the host (CPU only): one JSON line with the contract's keys
(impl, metric, value, unit, n_gpus, steps, warmup, ms_per_step, higher_is_better, scaling,
vs_baseline, dtype, data, config, cpu_baseline, e2e) -- the oracle timed on a bounded sample,
here over a small corpus so the test takes seconds."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3", "--n", "20000"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in j, key
    assert j["impl"] == "reference" and j["unit"] == "queries/s" and j["value"] > 0
    assert j["steps"] == 1 and j["warmup"] == 3 and j["higher_is_better"] is True
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["value"] == j["value"]
    assert "workload" in j["config"]


def test_bench_refuses_timing_experiment_switches():
    """SA_EXPERIMENT (and the other tuning switches) never reach a timed run: bench.py exits 2
    with an error line before loading anything."""
    env = dict(os.environ, SA_EXPERIMENT="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 2
    j = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert "SA_EXPERIMENT" in j["error"]


def test_bench_checks_world_size_against_gpus():
    """--gpus N under a launcher whose WORLD_SIZE differs is an error, never a silent 1-rank
    run."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=env)
    assert r.returncode == 2
    j = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert "WORLD_SIZE" in j["error"]


def test_bench_gpus_n_spawns_n_ranks():
    """`bench.py --gpus 2` without a launcher re-execs itself as 2 ranks under
    torch.distributed.run (127.0.0.1 rendezvous); checked here with a gloo group on CPU."""
    env = dict(os.environ, SA_BENCH_SPAWN_CHECK="1")
    for v in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(v, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0]) == {"spawn_check": 2, "ranks_seen": 2}
