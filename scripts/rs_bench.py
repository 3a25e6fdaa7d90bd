"""rs_adam in isolation through the C ABI (dc_reduce_scatter_step): one
Llama-3-8B-shaped layer (218 M shard elements at N = 1), LDG kernel vs the
bulk-copy pipelined kernel (option rs_bulk), CUDA events around each launch.
Algorithmic bytes per element at N virtual ranks: 2 N (grads) + 12 read +
12 write + 2 (bf16 shard) = 26 + 2N.

    python scripts/rs_bench.py [world] [reps]
"""
import ctypes as C
import dataclasses
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2504_09983_b200 import dc, runtime as rt  # noqa: E402


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    cfg = dataclasses.replace(synth.LLAMA3_8B, layers=2)
    table = synth.llama_param_table(cfg)
    ranks = rt.create_ranks(table, world, lr=1.5e-5, init=False)
    elems = ranks[0].layout.shard_elems // 2            # one layer
    for st in ranks.values():
        for k in ("master", "m", "v"):
            st.tensors[k].uniform_(0.0, 1e-3)
        st.tensors["grad"].view(torch.int16).random_(0, 16000)
    torch.cuda.synchronize()
    out = {"world": world, "elements": elems, "bytes_per_element": 26 + 2 * world}
    step = [0]

    def run(bulk):
        times = []

        def work(st):
            dc.check(dc.lib.dc_set_option(st.ctx, b"rs_bulk", bulk), st.ctx)
            cs, rs = st.streams[0], st.streams[2]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dc.check(dc.lib.dc_grad_slot_acquire(st.ctx, 0, cs.cuda_stream), st.ctx)
            dc.check(dc.lib.dc_grad_slot_publish(st.ctx, 0, cs.cuda_stream), st.ctx)
            ev = torch.cuda.Event()
            ev.record(cs)
            rs.wait_event(ev)
            e0.record(rs)
            dc.check(dc.lib.dc_reduce_scatter_step(st.ctx, 0, step[0], 0, rs.cuda_stream), st.ctx)
            e1.record(rs)
            torch.cuda.synchronize()
            if st.rank == 0:
                times.append(e0.elapsed_time(e1))

        for _ in range(reps):
            step[0] += 1
            rt.run_parallel(ranks, work)
        rt.poll(ranks)
        t = sorted(times[2:])[len(times[2:]) // 2]
        # per rank (virtual ranks share the GPU: at N > 1 the device total is N x this)
        return {"ms_median": t, "tb_s_per_rank": elems * (26 + 2 * world) / (t * 1e-3) / 1e12}

    if os.environ.get("RS_SERIAL"):
        # for ncu (kernels serialised): every rank publishes before any rank's
        # reduce-scatter waits, all from this thread
        bulk = int(os.environ.get("DC_RS_BULK", "0"))
        for t in (1, 2):
            for st in ranks.values():
                dc.check(dc.lib.dc_set_option(st.ctx, b"rs_bulk", bulk), st.ctx)
                dc.check(dc.lib.dc_grad_slot_acquire(st.ctx, 0, st.streams[0].cuda_stream), st.ctx)
                dc.check(dc.lib.dc_grad_slot_publish(st.ctx, 0, st.streams[0].cuda_stream), st.ctx)
            torch.cuda.synchronize()
            for st in ranks.values():
                dc.check(dc.lib.dc_reduce_scatter_step(st.ctx, 0, t, 0, st.streams[0].cuda_stream), st.ctx)
            torch.cuda.synchronize()
        rt.poll(ranks)
        return
    for _ in range(2):
        out["ldg"] = run(0)
        out["bulk"] = run(1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
