"""Config 3 plan study (BASELINE configs[2]): Llama-3-70B-shaped stack, L = 80,
N = 8, b = 1, seq 2048, with layer activation checkpointing, under a memory
budget sweep M in {155.7, 140, 130} GB — the prefetch vs selective-unshard
trade-off of PAPER.md §4.2-§4.3.  Host-only: one GPU cannot hold
an 8-rank 70B plan, so this runs dc_plan (the product planner, C ABI) on the
executor's S_0 with an analytic P_mem that mirrors model.cu's bookkeeping, and
times the schedules with the oracle's three-stream replay (oracle/sim.py,
reading D23) from per-op durations measured on the B200 (70B layers at N = 1,
profiles/r01g/lines_final/llama70b_L8.json) and an assumed T_c = 20 us + V / (0.7 x
900 GB/s).  Planning and memory numbers are exact; times are a model.

    python tests/tools/plan_sweep.py [--out profiles/r01g/plan_sweep_70b_n8.md]
"""
import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import sim  # noqa: E402
from tests.sched_util import analytic_profile as profile  # noqa: E402
from paper_2504_09983_b200 import dc  # noqa: E402

GB = 10 ** 9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01g", "plan_sweep_70b_n8.md"))
    ap.add_argument("--layers", type=int, default=80)
    args = ap.parse_args()
    N = 8
    cfg = dataclasses.replace(synth.LLAMA3_70B, layers=args.layers, seq=2048, batch=1)
    with open(os.path.join(ROOT, "profiles", "r01g", "lines_final", "llama70b_L8.json")) as fh:
        meas = json.load(fh)
    L_meas, b_meas = 8, 2
    # per layer, per op, at b = 1 (the measured run is 8 layers at b = 2)
    op_ms = {k: v / L_meas / b_meas for k, v in meas["kernels"]["op_ms_per_step"].items() if k != "rs"}
    bw = 0.7 * 900e3                      # bytes per us at 70 % of 900 GB/s
    tc = [[0, 20], [1 << 34, 20 + int((1 << 34) / bw)]]
    prof, E, B, layers = profile(cfg, N, op_ms)
    prof["tc"] = tc
    # RS of a layer: (N-1)/N of its gradient bytes in at 70 % of 900 GB/s + 20 us
    layer_bytes = {l: sum(B[i] for i in ids) for l, ids in layers.items()}
    for o in prof["ops"]:
        if o["kind"] == "rs":
            o["dur_us"] = 20 + int(layer_bytes[o["layer"]] * (N - 1) / N / bw)
    M_opt = 8 * E
    base_peak = max(o["p_mem"] for o in prof["ops"])
    rows = []
    for M_gb in (155.7, 140.0, 130.0):
        M = int(M_gb * GB)
        for name, passes in (("S0", dc.DC_PASS_SHARD), ("P", dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH),
                             ("S", dc.DC_PASS_SHARD | dc.DC_PASS_UNSHARD),
                             ("P+S", dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD)):
            t0 = time.perf_counter()
            try:
                h = dc.plan(json.dumps(prof), M, passes=passes, strict=True)
            except RuntimeError as e:
                rows.append((M_gb, name, "infeasible: %s" % str(e)[:60], "", "", "", ""))
                continue
            plan = json.loads(dc.schedule_json(h))
            dc.lib.dc_schedule_free(h)
            plan_ms = (time.perf_counter() - t0) * 1e3
            n_ag = sum(o["kind"] == "ag" for o in plan["ops"])
            unsh = set(plan["unshard"])
            unsh_layers = sum(1 for ids in layers.values() if set(ids) <= unsh)
            t_us = sim.simulate(plan["ops"], prof)
            peak = plan["peak_no_opt"] + M_opt
            rows.append((M_gb, name, "%.1f" % (float(t_us) / 1e3), len(unsh), unsh_layers, n_ag,
                         "%.1f / %.1f" % (peak / GB, plan["capacity"] / GB)))
    compute_ms = sum(o["dur_us"] for o in prof["ops"] if o["kind"] == "compute") / 1e3
    lines = ["# Config 3 plan study: Llama-3-70B-shaped, L = %d, N = 8, b = 1, seq 2048, layer checkpointing" % cfg.layers,
             "",
             "`python tests/tools/plan_sweep.py` (host-only; dc_plan = the product planner; times from the oracle's",
             "three-stream replay, reading D23).  Per-rank state %.1f GB (14 B x %.1f G shard elements), S_0 peak"
             % (14 * E / GB, E / 1e9),
             "without m/v %.1f GB; serial compute %.0f ms per step (per-op durations measured on B200, 70B layers at"
             % (base_peak / GB, compute_ms),
             "N = 1, profiles/r01g/lines_final/llama70b_L8.json, scaled to b = 1); T_c = 20 us + V / (0.7 x 900 GB/s)"
             " (model, not measured: one GPU).", "",
             "| M (GB) | passes | step (ms, replay) | unsharded params | unsharded layers | gathers / step | peak incl. m,v / arena (GB) |",
             "|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append("| %s |" % " | ".join(str(x) for x in r))
    lines += ["", "Reading: unshard ranks params by T_c(B)/B (P:364), so it keeps the latency-dominated small",
              "tensors first (norm gains, k/v: 16 KiB-16 MiB) and only then whole layers (1.71 GB each); a",
              "tighter M cuts the kept set (gathers per step rise back toward 1440).  Prefetch alone already hides",
              "most of the gather time in this replay (exposed communication = step - serial compute); with both",
              "passes the unshard pass removes gathers without hurting the prefetch."]
    out = "\n".join(lines) + "\n"
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        fh.write(out)
    print(out)


if __name__ == "__main__":
    main()
