"""bench.py end to end on the GPU (contract keys of the JSON line): N = 1 on a
2-layer stack, and the torchrun N = 2 flow (per-rank processes, peer maps,
flag protocol, profile MAX-reduce, identical plans) with both ranks sharing
cuda:0 (--share-gpu: its numbers are not bench values)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(out):
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and len(lines) == 1, out.stderr[-3000:]
    return json.loads(lines[0])


def _env():
    env = dict(os.environ)
    env["CUDA_DEVICE_MAX_CONNECTIONS"] = "8"     # processes sharing one GPU (see conftest.py)
    return env


def test_bench_n1_contract():
    out = subprocess.run([sys.executable, "bench.py", "--layers", "2", "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900, env=_env())
    d = _line(out)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] <= 1.2 and r["achieved_stream_ordered"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 4096 * 4096 * 2 and d["e2e"]["d2h_bytes_per_step"] == 4
    assert d["memory"]["device_peak_allocated"] > 0
    assert d["exposed_comm"]["frac"] is None and d["collectives"]["measured"] is False


def test_bench_self_launch_n2_share_gpu():
    """`bench.py --gpus 2` with no torchrun around it launches one process per
    rank itself (here both on cuda:0 with --share-gpu) and prints one line."""
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--layers", "2",
                          "--batch", "1", "--share-gpu"], cwd=ROOT, capture_output=True, text=True, timeout=900,
                         env={k: v for k, v in _env().items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")})
    d = _line(out)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "fsdp2"
    c = d["collectives"]
    assert c["measured"] and c["n_ranks"] == 2
    assert c["gathers_per_step"] > 0 and c["ag_busbw_gbs"] > 0 and c["rs_busbw_gbs"] > 0
    assert len(d["config"]["tc_table"]) >= 2
    assert d["exposed_comm"]["frac"] is not None
