"""T_c(V) sweep of our own all-gather (Table 1 / line
305, the Fuse rule at line 350) on one GPU: N virtual ranks (DC_VIRTUAL_RANKS,
every "peer" is another rank's buffer on the same device), full gathered sizes
V = 2^10 .. 2^max B, SM push kernel (ag_push) and copy-engine gathers
(option ag_copy_engine).  Through the C ABI only: a synthetic parameter table
with one parameter of each size (one layer each), an S_0 profile of gather /
consume / release per parameter, dc_plan (passes: shard), dc_bind_schedule,
then per step dc_step_begin + dc_gather / dc_release on every rank.

Each gather is timed on every rank's AG stream with the events of
dc_gather_timing: from "every receiver ready" to "every sender's stores landed
here" (the transfer time T_c the planner uses; the wait for the
receivers, which on one GPU is dominated by the Python threads' enqueue skew,
is excluded), max over ranks; median over steps.  On one GPU all N ranks' stores land in the same HBM, so the figure of
merit is the device's HBM traffic: every rank reads its shard once and writes
it into N arenas -> V (reads) + N V (writes) bytes per gather, against the
measured copy peak (MEASURED_PEAKS.json hbm_gbs, read + write).  The
NVLink-side busbw, (N-1)/N V / t, is what the same kernel delivers per GPU
on an NVSwitch box when NVLink, not HBM, is the bottleneck — it is reported
for the T_c table but is NOT an NVLink measurement.

    python scripts/ag_sweep.py [--worlds 2,4,8] [--max-log2 31] [--steps 5] [--out FILE]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import synth  # noqa: E402
from paper_2504_09983_b200 import dc, runtime as rt  # noqa: E402


def table_of(sizes):
    """One bf16 parameter of V/2 elements per size, parameter i in layer i."""
    return [synth.ParamSpec(id=i, layer=i, name="v%d" % v, shape=(v // 2,), k=0.0, dtype="bf16")
            for i, v in enumerate(sizes)]


def s0_profile(n, world, sizes):
    """S_0 of one forward region: ag(i), consume(i), rel(i) for every i, then a
    final compute op.  Ids = positions."""
    ops = []

    def add(kind, layer, params):
        ops.append({"id": len(ops), "kind": kind, "phase": "fwd", "micro": 0, "layer": layer, "params": params,
                    "p_mem": 0, "transient": 0, "dur_us": 0, "name": "use%d" % layer if kind == "compute" else kind})

    for i in range(n):
        add("ag", i, [i])
        add("compute", i, [i])
        add("rel", i, [i])
    add("compute", n - 1, [])
    S = [-(-(v // 2) // (8 * world)) * 8 for v in sizes]
    params = [{"id": i, "bytes": world * S[i] * 2, "layer": i} for i in range(n)]
    return {"ops": ops, "params": params, "frags": [], "tc": [[0, 0], [1 << 40, 0]]}


GATE = True


def sweep(world, sizes, steps, mode, hbm_peak):
    """mode: sm (16-byte stores), ce (copy engines), bulk (bulk-copy / TMA pipeline), chunked (fused_ag's
    chunk-ordered push with per-chunk flags)."""
    table = table_of(sizes)
    ranks = rt.create_ranks(table, world, init=False)
    for st in ranks.values():
        st.tensors["shard"].view(torch.int16).random_(-30000, 30000)
        dc.check(dc.lib.dc_set_option(st.ctx, b"ag_copy_engine", int(mode == "ce")), st.ctx)
        dc.check(dc.lib.dc_set_option(st.ctx, b"ag_bulk", int(mode == "bulk")), st.ctx)
        dc.check(dc.lib.dc_set_option(st.ctx, b"fused_ag", int(mode == "chunked")), st.ctx)
    prof = s0_profile(len(sizes), world, sizes)
    sched = dc.plan(json.dumps(prof), 1 << 50, passes=dc.DC_PASS_SHARD)
    plan = json.loads(dc.schedule_json(sched))
    rt.bind(ranks, {r: sched for r in ranks})
    ag = [o for o in plan["ops"] if o["kind"] == "ag"]
    rel = {o["members"][0]: o["id"] for o in plan["ops"] if o["kind"] == "rel"}
    times = {o["id"]: [] for o in ag}
    evs = {r: {o["id"]: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for o in ag}
           for r in ranks}
    for per in evs.values():             # torch creates the CUDA event at its first record
        for e0, e1 in per.values():
            e0.record()
            e1.record()

    gate_stream = torch.cuda.Stream()
    gate = {}

    def one_step(st, t):
        cs, ags = st.streams[0], st.streams[1]
        if GATE:
            cs.wait_event(gate["ev"])    # the device starts this step only after every rank enqueued it
        dc.check(dc.lib.dc_step_begin(st.ctx, t, cs.cuda_stream), st.ctx)
        for o in ag:
            e0, e1 = evs[st.rank][o["id"]]
            ev = torch.cuda.Event()
            ev.record(cs)
            ags.wait_event(ev)
            dc.check(dc.lib.dc_gather_timing(st.ctx, C.c_void_p(e0.cuda_event), C.c_void_p(e1.cuda_event)), st.ctx)
            dc.check(dc.lib.dc_gather(st.ctx, o["id"], ags.cuda_stream, None), st.ctx)
            cs.wait_event(e1)
            dc.check(dc.lib.dc_release(st.ctx, rel[o["members"][0]], cs.cuda_stream), st.ctx)
        torch.cuda.synchronize()

    for t in range(1, steps + 3):
        if GATE:      # a ~50 ms spin on a side stream holds every rank's step until all are enqueued, so
            with torch.cuda.stream(gate_stream):     # small gathers are not timed against host enqueue skew
                torch.cuda._sleep(int(50e-3 * 2e9))
                gate["ev"] = torch.cuda.Event()
                gate["ev"].record(gate_stream)
        rt.run_parallel(ranks, lambda st: one_step(st, t))
        rt.poll(ranks)
        if t > 2:                                   # two warm-up steps
            for o in ag:
                times[o["id"]].append(max(evs[r][o["id"]][0].elapsed_time(evs[r][o["id"]][1]) for r in ranks))
    rows = []
    for o, v in zip(ag, sizes):
        ms = statistics.median(times[o["id"]])
        full = o["bytes"]
        hbm = (world + 1) * full
        rows.append({"bytes": full, "us": ms * 1e3, "hbm_gbs": hbm / (ms * 1e-3) / 1e9,
                     "hbm_frac": hbm / (ms * 1e-3) / 1e9 / hbm_peak,
                     "busbw_gbs_if_nvlink": (world - 1) / world * full / (ms * 1e-3) / 1e9})
    del ranks
    torch.cuda.empty_cache()
    return rows


def push_only(world, sizes, reps=2, mode="sm"):
    """For ncu (kernels serialised: a flag wait on another rank's kernel would
    never return): rank 0 alone pushes each size with ag_skip_waits, so every
    ag_push launch runs by itself; nothing gathered this way is read."""
    table = table_of(sizes)
    ranks = rt.create_ranks(table, world, init=False)
    st = ranks[0]
    dc.check(dc.lib.dc_set_option(st.ctx, b"ag_skip_waits", 1), st.ctx)
    dc.check(dc.lib.dc_set_option(st.ctx, b"ag_bulk", int(mode == "bulk")), st.ctx)
    sched = dc.plan(json.dumps(s0_profile(len(sizes), world, sizes)), 1 << 50, passes=dc.DC_PASS_SHARD)
    plan = json.loads(dc.schedule_json(sched))
    rt.bind(ranks, {r: sched for r in ranks})
    dc.check(dc.lib.dc_step_begin(st.ctx, 1, st.streams[0].cuda_stream), st.ctx)
    for _ in range(reps):
        for o in plan["ops"]:
            if o["kind"] == "ag":
                dc.check(dc.lib.dc_gather(st.ctx, o["id"], st.streams[1].cuda_stream, None), st.ctx)
    torch.cuda.synchronize()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--max-log2", type=int, default=31)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ag_sweep.json"))
    ap.add_argument("--modes", default="sm,ce")
    ap.add_argument("--ncu-push", type=int, default=0, help="push-only run for ncu at this N (sizes >= 2^24)")
    ap.add_argument("--no-gate", action="store_true",
                    help="let each rank's step start as its host thread enqueues it (the r02 sweeps before the gate)")
    args = ap.parse_args()
    global GATE
    GATE = not args.no_gate
    if args.ncu_push:
        torch.cuda.set_device(0)
        push_only(args.ncu_push, [1 << k for k in range(24, args.max_log2 + 1, 2)], mode=args.modes.split(",")[0])
        return
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hbm_peak = json.load(fh)["hbm_gbs"]
    except (OSError, ValueError, KeyError):
        hbm_peak = 6546.6
    torch.cuda.set_device(0)
    sizes = [1 << k for k in range(10, args.max_log2 + 1)]
    out = {"hbm_peak_gbs": hbm_peak, "note": __doc__.split("\n\n")[1], "runs": []}
    for world in [int(w) for w in args.worlds.split(",")]:
        for mode in args.modes.split(","):
            rows = sweep(world, sizes, args.steps, mode, hbm_peak)
            out["runs"].append({"world": world, "mode": mode, "rows": rows,
                                "tc_table": [[r["bytes"], max(1, int(round(r["us"])))] for r in rows]})
            big = [r for r in rows if r["bytes"] >= (64 << 20)]
            print("N=%d %s: >=64MiB HBM %.0f GB/s (%.2f of peak); 1 KiB %.1f us" %
                  (world, mode, statistics.mean(r["hbm_gbs"] for r in big) if big else 0,
                   statistics.mean(r["hbm_frac"] for r in big) if big else 0, rows[0]["us"]), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
