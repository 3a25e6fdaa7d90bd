"""Gradient-accumulation plan study at N = 8 (§5.3: the
paper's largest gains, 1.28x / 1.54x over ZeRO-3, are at GA 16 where selective
unsharding keeps parameters gathered across micro-steps).  Host-only: dc_plan
(the product planner) on full-size S_0 profiles with n micro-steps
(tests/sched_util.analytic_profile), timed by the oracle's three-stream replay
(reading D23) with per-op durations measured on the B200 at N = 1 and an
assumed T_c = 20 us + V / (0.7 x 900 GB/s).  S_0 (gather before every use,
release after: no prefetch, no unshard) is the ZeRO-3-like baseline of the
same executor; P+S is DeepCompile's schedule.  Plans and memory are exact;
times are a model.

    python tests/tools/ga_sweep.py [--out profiles/r01g/ga_sweep_n8.md]
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
from paper_2504_09983_b200 import dc  # noqa: E402
from tests.sched_util import analytic_profile  # noqa: E402

GB = 10 ** 9


def per_op_ms(path, layers, batch):
    """Measured per-op ms (N = 1 bench line), per layer and per op name, scaled to b = 1."""
    with open(os.path.join(ROOT, path)) as fh:
        meas = json.load(fh)
    acc = {}
    for k, v in meas["kernels"]["op_ms_per_step"].items():
        if k == "rs":
            continue
        head, _, tail = k.rpartition("_")
        base = head if tail.isdigit() else k
        acc.setdefault(base, []).append(v / layers / batch)
    return {k: sum(v) / len(v) for k, v in acc.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01g", "ga_sweep_n8.md"))
    args = ap.parse_args()
    N = 8
    bw = 0.7 * 900e3
    tc = [[0, 20], [1 << 34, 20 + int((1 << 34) / bw)]]
    models = [("Mixtral-8x7B L = 32", synth.MIXTRAL_8X7B, 32, per_op_ms("profiles/r01g/lines_final/mix_b2.json", 4, 2)),
              ("Llama-3-8B L = 32", synth.LLAMA3_8B, 32, per_op_ms("profiles/r01g/bench_default_final.json", 32, 2))]
    rows = []
    for label, base, L, op_ms in models:
        cfg = dataclasses.replace(base, layers=L, seq=2048, batch=1)
        for n in (1, 4, 16):
            prof, E, B, layers = analytic_profile(cfg, N, op_ms, checkpoint=False, micro_steps=n)
            prof["tc"] = tc
            layer_bytes = {l: sum(B[i] for i in ids) for l, ids in layers.items()}
            for o in prof["ops"]:
                if o["kind"] == "rs":
                    o["dur_us"] = 20 + int(layer_bytes[o["layer"]] * (N - 1) / N / bw)
            compute_ms = sum(o["dur_us"] for o in prof["ops"] if o["kind"] == "compute") / 1e3
            M = int(155.7 * GB)
            res = {}
            for name, passes in (("S0", dc.DC_PASS_SHARD), ("P", dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH),
                                 ("P+S", dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD)):
                t0 = time.perf_counter()
                h = dc.plan(json.dumps(prof), M, passes=passes, strict=True)
                plan = json.loads(dc.schedule_json(h))
                dc.lib.dc_schedule_free(h)
                t_plan = time.perf_counter() - t0
                ms = float(sim.simulate(plan["ops"], prof)) / 1e3
                res[name] = (ms, sum(o["kind"] == "ag" for o in plan["ops"]), len(plan["unshard"]), t_plan)
            tokens = N * cfg.tokens * n
            rows.append((label, n, len(prof["ops"]), compute_ms, res, tokens))
            print(label, n, {k: round(v[0], 1) for k, v in res.items()}, flush=True)
    lines = ["# Gradient accumulation at N = 8: S_0 (ZeRO-3-like) vs prefetch vs prefetch + selective unshard",
             "",
             "`python tests/tools/ga_sweep.py` (host-only; dc_plan on full-size S_0 profiles with n micro-steps; oracle",
             "three-stream replay, D23; per-op durations measured on B200 at N = 1 (profiles/r01g), b = 1, seq 2048;",
             "T_c = 20 us + V / (0.7 x 900 GB/s), RS(l) = (N-1)/N of the layer's bytes at the same rate; M = 155.7 GB).",
             "Times are a model; the plans (gathers, unsharded parameters) are the planner's exact output.", "",
             "| model | GA n | S_0 ops | serial compute (ms) | S_0 step (ms) / gathers | P step / gathers | P+S step / gathers / unsharded | P+S vs S_0 | P+S tokens/s/box |",
             "|---|---|---|---|---|---|---|---|---|"]
    for label, n, nops, comp, res, tokens in rows:
        s0, p, ps = res["S0"], res["P"], res["P+S"]
        lines.append("| %s | %d | %d | %.0f | %.0f / %d | %.0f / %d | %.0f / %d / %d | %.2fx | %.0f |" % (
            label, n, nops, comp, s0[0], s0[1], p[0], p[1], ps[0], ps[1], ps[2], s0[0] / ps[0],
            tokens / (ps[0] / 1e3)))
    lines += ["", "Context (not a target): the paper reports 1.28x (Llama-3 70B) and 1.54x (Mixtral 8x7B) over",
              "ZeRO-3 at GA 16 on its H100 cluster (P:474-478).  S_0 here has no prefetch at all (each gather waits",
              "for the preceding compute op, reading D23), while ZeRO-3 has its own bucketed prefetcher, so these",
              "ratios overstate that comparison.  The gain grows with n because the unshard pass keeps the",
              "selected parameters gathered across all n micro-steps (2 gathers per step instead of 2n), while",
              "prefetch alone only hides each gather behind the previous op's compute.  At Llama-3-8B size every",
              "parameter fits gathered (288 unsharded), so P+S issues one gather per parameter per step."]
    out = "\n".join(lines) + "\n"
    with open(args.out, "w") as fh:
        fh.write(out)
    print(out)


if __name__ == "__main__":
    main()
