"""Per-op CUDA-event times of one profiled step (diagnostic): python
scripts/op_times.py [model] [layers] [batch].  Prints the per-op-name sums and
the first layer's forward sequence (DC_OPT_BWD=1: also the backward sequence
of the last and the first layer; DC_OPT_PASSES: plan passes, default S_0)."""
import dataclasses
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2504_09983_b200 import dc, runtime as rt  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "MIXTRAL_8X7B"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
b = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = dataclasses.replace(getattr(synth, name), layers=L, batch=b)
table = synth.param_table(cfg)
ranks = rt.create_ranks(table, 1, lr=1e-5)
st = ranks[0]
T = cfg.tokens
x = torch.randn(T, cfg.hidden, device="cuda").to(torch.bfloat16)
t = torch.randn(T, cfg.hidden, device="cuda").to(torch.bfloat16)
rt.attach_model(ranks, cfg, {0: x}, {0: t})
for k, v in os.environ.items():
    if k.startswith("DCOPT_"):
        dc.check(dc.lib.dc_model_set_option(st.model, k[6:].lower().encode(), int(v)))
prof = rt.profile_json(st)
passes = int(os.environ.get("DC_OPT_PASSES", dc.DC_PASS_SHARD))
rt.bind(ranks, {0: dc.plan(json.dumps(prof), 1 << 50, passes=passes)})
for s in range(1, 4):
    rt.step(ranks, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st.streams[0])
rt.step(ranks, 4, profile=1)
e1.record(st.streams[0])
torch.cuda.synchronize()
print("step ms", e0.elapsed_time(e1))
p = json.loads(dc.model_profile_json(st.model))
agg = {}
for o in p["ops"]:
    if o["kind"] in ("compute", "rs"):
        agg[o["name"]] = agg.get(o["name"], 0) + o["dur_us"]
print(json.dumps({k: v / 1e3 for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:25]}))
print([(o["name"], o["dur_us"]) for o in p["ops"] if o["kind"] == "compute" and o["layer"] == 0 and o["phase"] == "fwd"])
if os.environ.get("DC_OPT_BWD"):
    for l in (L - 1, 0):
        print("bwd layer", l, [(o["kind"], o["name"], o["dur_us"]) for o in p["ops"]
                               if o["layer"] == l and o["phase"] == "bwd"])
