"""CPU: bench.py's multi-GPU launch path.  `bench.py --gpus 2` outside torchrun
re-runs itself as 2 ranks (torch.distributed.run on 127.0.0.1, one process per
GPU); --dry-run keeps the ranks on CPU (gloo) so the launcher, the unit shards
and the max-over-ranks reduction are exercised without a GPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["NCCL_DEBUG_FILE"] = os.devnull
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_self_launch_two_ranks_weak():
    j = _run("--gpus", "2", "--dry-run", "--steps", "4", "--warmup", "3")
    assert j["n_gpus"] == 2 and j["dry_run"]
    assert j["scaling"] == "weak"
    # weak scaling: every rank serves its own batch of 64 x 32 units
    assert j["units_per_rank"] == [2048, 2048]
    assert j["config"]["global_batch"] == 128
    assert j["max_rank_time_s"] == 2e-3  # max over ranks, not rank 0's own


def test_self_launch_two_ranks_strong_c5():
    j = _run("--gpus", "2", "--dry-run", "--config", "c5", "--steps", "4", "--warmup", "3")
    assert j["n_gpus"] == 2 and j["scaling"] == "strong"
    # strong scaling: the 16 x 32 units of C5 are split, batch-major
    assert j["units_per_rank"] == [256, 256]
    assert j["config"]["global_batch"] == 16


def test_single_rank_dry_run():
    j = _run("--dry-run", "--steps", "4", "--warmup", "3")
    assert j["n_gpus"] == 1 and j["units_per_rank"] == [2048]


def test_reference_arm_config_matches_ours():
    """Both arms report the same config dict for the same arguments (the
    driver compares them)."""
    sys.path.insert(0, ROOT)
    import importlib
    bench = importlib.import_module("bench")
    import argparse
    a = argparse.Namespace(config="c2", layers=0, bits=0, scaling=None, steps=20, warmup=5,
                           gpus=1)
    c1, u1, s1 = bench.workload_config(a, 1, 0, None)
    c2, u2, s2 = bench.workload_config(a, 1, 0, 180e9)
    assert c1 == c2 and u1 == u2 == 2048 and s1 == s2 == "weak"


def test_clock_rejection_rule():
    """bench.py re-measures once when the timed region saw a hardware / thermal
    slowdown or clocks stuck well below max with no reason; a power cap is kept."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    ok = {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": []}
    assert not bench.clocks_bad(ok)
    assert not bench.clocks_bad(dict(ok, sm_mhz=1700, reasons=["sw_power_cap"]))
    assert bench.clocks_bad(dict(ok, reasons=["hw_slowdown"]))
    assert bench.clocks_bad(dict(ok, reasons=["sw_power_cap", "sw_thermal_slowdown"]))
    assert bench.clocks_bad(dict(ok, sm_mhz=1200))
    assert not bench.clocks_bad({"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]})
