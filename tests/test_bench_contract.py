"""bench.py's reference arm keeps the driver's JSON contract (CPU only).

`bench.py --impl reference` times the reference's own CPU implementation
(oracle/_ref, else the C port) and prints one JSON line with the contract's
keys; under torchrun only rank 0 prints, the other ranks exit 0 without work.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(extra_env=None):
    env = dict(os.environ, OMP_NUM_THREADS="2", **(extra_env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--config", "c1", "--steps", "2", "--warmup", "1"],
                          capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)


def test_reference_arm_json_line():
    r = run()
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "iter/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["steps"] == 2
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1 and cb["kind"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 == e["d2h_bytes_per_step"]
    assert d["config"]["workload"] and "model" not in d["config"]


def test_reference_arm_other_ranks_silent():
    r = run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """The headline arm on a GPU: every key the driver reads, with the kernel
    roofline, the CPU baseline, the end-to-end number and the launch count."""
    try:
        import torch
        if not torch.cuda.is_available():
            pytest.skip("no GPU")
    except Exception:
        pytest.skip("no torch")
    env = dict(os.environ, OMP_NUM_THREADS="4")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1",
                        "--steps", "5", "--warmup", "3", "--cpu-iters", "2"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip()][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 5 and d["warmup"] == 3 and d["n_gpus"] == 1
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["achieved"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    # two sweeps per iteration at least (C1: consumed reductions)
    assert d["gpu_launches"] >= 2 * d["steps"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
@pytest.mark.parametrize("n,config", [(2, "c1"), (4, "c1")])
def test_gpu_arm_multi_rank_reexec(n, config):
    """`python bench.py --gpus N` outside torchrun relaunches itself as N ranks
    (here all on GPU 0: ACG_SAME_GPU=1, peer-memory transport), reports
    n_gpus = N and verifies the N-rank residual history against the same
    iterations on one GPU, bit for bit (the slabs are reduction-tree nodes)."""
    try:
        import torch
        if not torch.cuda.is_available():
            pytest.skip("no GPU")
    except Exception:
        pytest.skip("no torch")
    env = dict(os.environ, OMP_NUM_THREADS="2", ACG_SAME_GPU="1")
    env.pop("WORLD_SIZE", None)
    # the 2-rank run also times the e2e stream (async transfers on every rank)
    extra = [] if n == 2 else ["--no-e2e"]
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                        "--config", config, "--steps", "5", "--warmup", "3", "--no-cpu",
                        "--sustain-steps", "20"] + extra,
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["exact_tree"] is True
    v = d["verified_vs_1gpu"]
    assert v["ok"] is True and v["exact_tree"] is True and v["max_dev_over_r0"] == 0.0
    assert d["sustained"]["steps"] == 20 and d["sustained"]["value"] > 0
    if n == 2:
        e = d["e2e"]
        assert e["value"] > 0 and e["solves"] >= 2 and e["serial"]["value"] > 0


@pytest.mark.gpu
def test_gpu_arm_long_small_grid_passes_restart():
    """Each measured pass restarts the solve: at C1 (whose residual reaches exactly
    zero after ~1400 iterations) a 1000-step run with the per-launch timing pass
    and a 1000-step sustained pass is valid; a single 3000-step pass is refused."""
    try:
        import torch
        if not torch.cuda.is_available():
            pytest.skip("no GPU")
    except Exception:
        pytest.skip("no torch")
    base = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--warmup", "3",
            "--no-cpu", "--no-e2e"]
    r = subprocess.run(base + ["--steps", "1000", "--sustain-steps", "1000"], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip()][-1])
    assert d["steps"] == 1000 and d["sustained"]["steps"] == 1000 and d["roofline"]["achieved"] > 0
    r = subprocess.run(base + ["--steps", "3000", "--sustain-steps", "0", "--no-ktime"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode != 0 and "converged" in (r.stdout + r.stderr)
