"""Diagnostic: run the smoke configuration with a short flag timeout and dump
both virtual ranks' flag tables (ready / done counters) if a wait times out."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from oracle import numerics as nx  # noqa: E402
from oracle import step as ost  # noqa: E402
from paper_2504_09983_b200 import dc, runtime as rt  # noqa: E402

seq = int(sys.argv[1]) if len(sys.argv) > 1 else 128
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 7
cfg = synth.small_llama(layers=2, seq=seq)
table = synth.llama_param_table(cfg)
ranks = rt.create_ranks(table, 2, lr=1e-3, spin_ms=3000)
xs, ts = {}, {}
for r in ranks:
    x, t = ost.rank_batch(cfg, r)
    xs[r] = torch.from_numpy(nx.bf16_bits(x).view(np.int16).copy()).cuda().view(torch.bfloat16)
    ts[r] = torch.from_numpy(nx.bf16_bits(t).view(np.int16).copy()).cuda().view(torch.bfloat16)
rt.attach_model(ranks, cfg, xs, ts)
prof = rt.profile_json(ranks[0], tc=[[4096, 10], [1 << 20, 20], [1 << 26, 400]])
sched = dc.plan(json.dumps(prof), 1 << 40, M_prefetch=1 << 22, passes=passes, strict=True)
plan = json.loads(dc.schedule_json(sched))
rt.bind(ranks, {r: sched for r in ranks})
ok = True
try:
    rt.step(ranks, 1)
    torch.cuda.synchronize()
    rt.poll(ranks)
except dc.DCError as e:
    ok = False
    print("ERROR", e)
torch.cuda.synchronize()
world = 2
mops = rt.max_s0_ops(table)
for r, st in ranks.items():
    f = st.tensors["flags"].view(torch.int32).cpu().numpy()
    ready = f[:mops * world].reshape(mops, world)
    done = f[mops * world: mops * world + mops]
    print("rank", r, "ok" if ok else "")
    for o in plan["ops"]:
        if o["kind"] == "ag":
            print("  ag %4d members %s waits %s ready %s done %d" % (o["id"], o["members"], o["waits_on"],
                                                                  ready[o["id"]].tolist(), done[o["id"]]))
print(json.dumps([o for o in plan["ops"] if o["kind"] in ("ag", "rel")])[:3000])
