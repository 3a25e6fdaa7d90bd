"""One planned N = 1 step of a one-layer Llama-shaped model at a chosen hidden
size, for compute-sanitizer runs of kernels whose launch shape depends on H
(the one-pass RMSNorm backward: G = H / 1024 warps per row at V = 4, named
barriers for G > 1).  No oracle (the -m gpu tests check the numbers).

    compute-sanitizer --tool racecheck python scripts/sanitize_step.py 2048
"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2504_09983_b200 import dc, runtime as rt  # noqa: E402


def main(hidden):
    heads = hidden // 128
    cfg = dataclasses.replace(synth.small_llama(layers=1, seq=40), hidden=hidden, ffn=256, n_heads=heads,
                              n_kv=max(2, heads // 4))
    table = synth.llama_param_table(cfg)
    ranks = rt.create_ranks(table, 1, lr=1e-3)
    n = cfg.tokens * cfg.hidden
    x = synth.values(synth.seed_inputs(0), 0, 0, n, synth.K_UNIT).astype(np.float32)
    t = synth.values(synth.seed_targets(0), 0, 0, n, synth.K_UNIT).astype(np.float32)
    rt.attach_model(ranks, cfg, {0: torch.from_numpy(x).cuda().bfloat16()}, {0: torch.from_numpy(t).cuda().bfloat16()})
    sched = dc.plan(json.dumps(rt.profile_json(ranks[0])), 1 << 40, passes=dc.DC_PASS_SHARD, strict=True)
    rt.bind(ranks, {0: sched})
    rt.step(ranks, 1)
    torch.cuda.synchronize()
    rt.poll(ranks)
    print("sanitize_step: H = %d, one step ok, loss %.6f" %
          (hidden, rt.view(rt.loss_ptr(ranks[0]), 1, torch.float32).item()))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2048)
