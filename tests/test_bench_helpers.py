"""bench.py's host-side helpers (CPU): the T_c table built from profiled
gathers, and the per-op GEMM FLOP accounting behind roofline.achieved."""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402


def test_tc_from_profile_median_sorted_monotone():
    prof = {"params": [{"id": 0, "bytes": 100}, {"id": 1, "bytes": 5000}, {"id": 2, "bytes": 100}],
            "ops": [{"kind": "ag", "params": [0], "dur_us": 30}, {"kind": "ag", "params": [2], "dur_us": 10},
                    {"kind": "ag", "params": [0], "dur_us": 20}, {"kind": "ag", "params": [1], "dur_us": 15},
                    {"kind": "ag", "params": [1], "dur_us": 0}, {"kind": "compute", "params": [0], "dur_us": 99}]}
    # size 100: median of 30, 10, 20 = 20; size 5000: 15 -> raised to 20 (non-decreasing)
    assert bench.tc_from_profile(prof) == [[100, 20], [5000, 20]]
    assert bench.tc_from_profile({"params": [], "ops": []}) is None


def test_gemm_flops_llama_and_moe():
    cfg = dataclasses.replace(synth.LLAMA3_8B, layers=1, seq=2048, batch=2)
    T, h, f = cfg.tokens, cfg.hidden, cfg.ffn
    assert bench.gemm_flops("gate_up", cfg, T) == 2 * T * h * 2 * f
    assert bench.gemm_flops("gate_up_bwd", cfg, T) == 4 * T * h * 2 * f
    assert bench.gemm_flops("re_qkv", cfg, T) == bench.gemm_flops("qkv", cfg, T)
    assert bench.gemm_flops("o_bwd", cfg, T) == 2 * bench.gemm_flops("o_proj", cfg, T)
    assert bench.gemm_flops("act", cfg, T) is None and bench.gemm_flops("rs", cfg, T) is None
    # a step's GEMM FLOPs = 6 x params x tokens for the Llama layer's matrices
    ops = ["qkv", "o_proj", "gate_up", "down", "qkv_bwd", "o_bwd", "gate_up_bwd", "down_bwd"]
    mats = sum(p.numel for p in synth.param_table(cfg) if not p.name.endswith("norm"))
    assert sum(bench.gemm_flops(o, cfg, T) for o in ops) == 6 * mats * T
    moe = dataclasses.replace(synth.MIXTRAL_8X7B, layers=1, seq=2048, batch=2)
    R = 2 * moe.tokens // moe.n_experts
    assert bench.gemm_flops("exp_gu_5", moe, moe.tokens) == 2 * R * moe.hidden * 2 * moe.ffn
    assert bench.gemm_flops("exp_down_bwd_0", moe, moe.tokens) == 4 * R * moe.ffn * moe.hidden


def test_load_tc_table_from_sweep_and_list(tmp_path):
    """--tc-table: an ag_sweep.py run (median us per size) or a plain [[bytes, us]] list ->
    integer, size-sorted, non-decreasing T_c table (the form dc_plan takes)."""
    import json

    import bench
    sweep = {"runs": [{"world": 8, "mode": "sm", "rows": [{"bytes": 4096, "us": 30.4}, {"bytes": 1024, "us": 41.2},
                                                         {"bytes": 1 << 20, "us": 55.6}]},
                      {"world": 2, "mode": "sm", "rows": [{"bytes": 1024, "us": 1.0}]}]}
    p = tmp_path / "sweep.json"
    p.write_text(json.dumps(sweep))
    assert bench.load_tc_table(str(p) + ":8:sm") == [[1024, 41], [4096, 41], [1 << 20, 56]]
    q = tmp_path / "list.json"
    q.write_text(json.dumps([[2048, 9], [1024, 5]]))
    assert bench.load_tc_table(str(q)) == [[1024, 5], [2048, 9]]
