"""bench.py's CPU-only arms (the driver runs `bench.py --impl reference`):
the oracle reference arm prints one JSON line with the contract keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_default_workload():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["unit"] == "tokens/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["config"]["layers"] == 32
    # ms_per_step is the sample actually timed (one layer sample), not an extrapolation
    assert d["ms_per_step"] < d["extrapolated_ms_per_workload_step"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_other_models_unavailable():
    d = _run("--impl", "reference", "--model", "mixtral-8x7b")
    assert d["impl"] == "reference" and "unavailable" in d


def test_self_launch_forks_ranks():
    """--gpus N outside torchrun re-launches itself with one process per rank
    (torch.distributed.run on 127.0.0.1) and passes rank 0's one JSON line
    through; --dry-run keeps the GPU out (gloo barrier + MAX over ranks)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    d = _run("--gpus", "2", "--dry-run", env=env)
    assert d["dry_run"] and d["n_gpus"] == 2
    assert sorted(d["ranks"]) == [0, 1] and d["processes"] == 2
    assert d["max_over_ranks"] == 2.0
