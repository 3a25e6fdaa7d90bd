"""Fused all-gather -> GEMM A/B on one GPU: N virtual ranks of
a Llama-3-8B-shaped stack, the same GEMM SM cap for both arms (1/N of the SMs
each, what fused mode needs for co-residency; DC_GEMM_SMS for the plain arm),
S_0 schedule (every gather issued right before its first consumer, so the
gather is on the critical path — what the fused GEMM attacks) and the planned
P+S schedule.  Device-timed steps (CUDA events on rank 0's compute stream
after a device-wide synchronize on both sides).  One JSON line per arm.

    python scripts/fused_ab.py [--world 2] [--layers 4] [--batch 1] [--steps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--fused", type=int, default=1)
    ap.add_argument("--passes", default="S0")
    a = ap.parse_args()
    import dataclasses

    import numpy as np
    import torch

    import synth
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    os.environ["DC_GEMM_SMS"] = str(max(2, sms // a.world // 2 * 2))     # read once by the library
    from paper_2504_09983_b200 import dc, runtime as rt
    cfg = dataclasses.replace(synth.LLAMA3_8B, layers=a.layers, batch=a.batch)
    table = synth.param_table(cfg)
    ranks = rt.create_ranks(table, a.world, lr=1.5e-5)
    for st in ranks.values():
        dc.check(dc.lib.dc_set_option(st.ctx, b"fused_ag", a.fused), st.ctx)
    T = cfg.tokens
    xs, ts = {}, {}
    for r in ranks:
        x = synth.values(synth.seed_inputs(r, 0), 0, 0, T * cfg.hidden, synth.K_UNIT)
        t = synth.values(synth.seed_targets(r, 0), 0, 0, T * cfg.hidden, synth.K_UNIT)
        xs[r] = torch.from_numpy(x).to(torch.bfloat16).cuda().view(T, cfg.hidden)
        ts[r] = torch.from_numpy(t).to(torch.bfloat16).cuda().view(T, cfg.hidden)
    rt.attach_model(ranks, cfg, xs, ts)
    for st in ranks.values():       # the plain arm: no second GEMM stream either (as fused mode)
        dc.check(dc.lib.dc_model_set_option(st.model, b"dw_concurrent", 0))
        dc.check(dc.lib.dc_model_set_option(st.model, b"stream_k", 0))
    prof = rt.profile_json(ranks[0], tc=[[1024, 30], [1 << 20, 40], [1 << 30, 40 + (1 << 30) // 4000]])
    passes = dc.DC_PASS_SHARD if a.passes == "S0" else \
        dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD
    sched = dc.plan(json.dumps(prof), 150 << 30, passes=passes, strict=True)
    rt.bind(ranks, {r: sched for r in ranks})
    step = 0
    for _ in range(3):
        step += 1
        rt.step(ranks, step)
        torch.cuda.synchronize()
        rt.poll(ranks)
    cs = ranks[0].streams[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(a.steps):
        step += 1
        torch.cuda.synchronize()
        e0.record(cs)
        rt.step(ranks, step)
        e1.record(cs)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    rt.poll(ranks)
    step += 1                                            # one profiled step: per-op event times
    rt.step(ranks, step, profile=True)
    torch.cuda.synchronize()
    prof = json.loads(dc.model_profile_json(ranks[0].model))
    ops = {}
    for o in prof["ops"]:
        if o["kind"] in ("compute", "rs", "ag"):
            k = o["kind"] if o["kind"] != "compute" else o.get("name", "?")
            ops[k] = round(ops.get(k, 0) + o["dur_us"] / 1e3, 3)
    print(json.dumps({"op_ms": ops, "world": a.world, "fused": a.fused, "passes": a.passes, "layers": a.layers,
                      "tokens_per_rank": T, "gemm_sms": int(os.environ["DC_GEMM_SMS"]),
                      "ms_per_step_median": float(np.median(ms)), "ms": ms}), flush=True)


if __name__ == "__main__":
    main()
