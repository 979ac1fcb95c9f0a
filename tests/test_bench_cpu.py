"""bench.py contract on CPU: the reference arm (the oracle port on host cores)
prints one JSON line with every key the driver reads, on the same workload
config object as the GPU arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--config", "c1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "ASADMM iterations/s" and d["unit"] == "iterations/s"
    assert d["higher_is_better"] is True and d["value"] > 0 and d["steps"] >= 1
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] in ("port", "reference")
    assert cb["value"] == d["value"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0
    cfg = d["config"]
    assert cfg["workload"].startswith("BASELINE c1:") and {"global_batch", "parallelism", "hyper"} <= set(cfg)
    assert cb["extrapolated"] is False  # config 1 fits: every sensor timed, no extrapolation


def test_workload_config_matches_between_arms():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2307_08606_b200 import scenario
    cfg = scenario.baseline_config("c2")
    ours = bench.workload_config(cfg, 1, 145.87408026212287)
    ref = bench.workload_config(cfg, 1, 145.87408026212301)  # the host's lambda: last-bit differences only
    assert ours == ref  # identical config objects (the driver's same_config check)
    assert bench.algorithmic_bytes_per_iteration(cfg, [cfg.N] * cfg.Q) > 4.5e9


def test_default_headline_config_is_c3():
    """python bench.py --gpus 1 prints the largest single-GPU BASELINE config
    (config 3, 171 GB resident), fixed iterations."""
    sys.path.insert(0, ROOT)
    import bench
    saved = sys.argv
    sys.argv = ["bench.py"]
    try:
        args = bench.parse()
    finally:
        sys.argv = saved
    assert args.config == "c3" and args.gpus == 1 and args.steps + args.warmup == 500


def test_gpus_flag_spawns_ranks_outside_torchrun(monkeypatch):
    """--gpus N without WORLD_SIZE re-launches through torch.distributed.run."""
    sys.path.insert(0, ROOT)
    import bench
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd, env=None: calls.append(cmd) or 0)

    class A:
        gpus = 4
    assert bench.spawn_ranks(A()) is True
    cmd = calls[0]
    assert "torch.distributed.run" in cmd and "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    A.gpus = 1
    assert bench.spawn_ranks(A()) is False
