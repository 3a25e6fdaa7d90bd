"""Adaptive offload (§4.4, Algorithm 2 + reload rule) on the
GPU path, with DC_DEBUG_POISON: once a fragment's D2H copy is synced the
device slice is overwritten with NaNs, so a missing or misordered reload
corrupts the Adam update.  The offloaded step must be bit-identical to the
same step without offload."""
import ctypes as C
import json

import numpy as np
import pytest
import torch

import synth
from oracle import step as ost
from tests.gpu_util import bf16_tensor

pytestmark = pytest.mark.gpu

dc = pytest.importorskip("paper_2504_09983_b200.dc")
from paper_2504_09983_b200 import runtime as rt  # noqa: E402

LR = 1e-3


def _ranks(cfg, world, poison):
    table = synth.llama_param_table(cfg)
    n = sum(-(-p.numel // (8 * world)) * 8 for p in table)
    ranks = rt.create_ranks(table, world, lr=LR, host_pinned_bytes=8 * n + 4096,
                            extra_flags=dc.DC_DEBUG_POISON if poison else 0)
    xs, ts = {}, {}
    for r in ranks:
        x, t = ost.rank_batch(cfg, r)
        xs[r], ts[r] = bf16_tensor(x), bf16_tensor(t)
    rt.attach_model(ranks, cfg, xs, ts)
    return table, ranks


def test_offload_op_roundtrip_with_poison():
    cfg = synth.small_llama(layers=2, seq=128)
    table, ranks = _ranks(cfg, 1, poison=True)
    st = ranks[0]
    frags = rt.offload_fragments(st, 64 * 1024)
    assert len(frags) >= 8 and all(f["bytes"] <= 64 * 1024 for f in frags)
    st.tensors["m"].uniform_(-1, 1)
    before = st.tensors["m"].clone()
    f0 = next(i for i, f in enumerate(frags) if f["layer"] == 1)
    cs, cp = st.streams[0].cuda_stream, st.streams[3].cuda_stream
    dc.check(dc.lib.dc_offload(st.ctx, f0, dc.DC_D2H_START, cp), st.ctx)
    dc.check(dc.lib.dc_offload(st.ctx, f0, dc.DC_D2H_SYNC_FREE, cs), st.ctx)
    torch.cuda.synchronize()
    assert torch.isnan(st.tensors["m"]).any()                 # poisoned after the free
    dc.check(dc.lib.dc_offload(st.ctx, f0, dc.DC_H2D_START, cp), st.ctx)
    dc.check(dc.lib.dc_offload(st.ctx, f0, dc.DC_H2D_SYNC, cs), st.ctx)
    torch.cuda.synchronize()
    assert torch.equal(st.tensors["m"].view(torch.int32), before.view(torch.int32))
    assert dc.lib.dc_offload(st.ctx, len(frags), dc.DC_D2H_START, cp) == dc.DC_EINVAL


@pytest.mark.parametrize("world", [1, 2])
def test_offload_step_bitexact_vs_resident(world):
    cfg = synth.small_llama(layers=2, seq=128)
    _, ref = _ranks(cfg, world, poison=False)
    prof = rt.profile_json(ref[0])
    s0 = dc.plan(json.dumps(prof), 1 << 40, passes=dc.DC_PASS_SHARD)
    rt.bind(ref, {r: s0 for r in ref})
    table, off = _ranks(cfg, world, poison=True)
    frags = None
    for st in off.values():
        frags = rt.offload_fragments(st, 128 * 1024)
    prof = rt.profile_json(off[0], frags=frags)
    peak = max(o["p_mem"] + o["transient"] for o in prof["ops"])
    m_opt = sum(f["bytes"] for f in frags)
    sched = dc.plan(json.dumps(prof), peak + m_opt // 2, passes=dc.DC_PASS_SHARD | dc.DC_PASS_OFFLOAD,
                    strict=True)
    plan = json.loads(dc.schedule_json(sched))
    kinds = [o["kind"] for o in plan["ops"]]
    assert plan["offload"] and kinds.count("offload") == len(plan["offload"])
    assert kinds.count("reload") == kinds.count("reload_sync") == kinds.count("offload_sync") == len(plan["offload"])
    rt.bind(off, {r: sched for r in off})
    if world == 1:   # fused Adam is requested on both; the offloading step must fall back to rs_adam
        for st in list(ref.values()) + list(off.values()):
            dc.check(dc.lib.dc_model_set_option(st.model, b"fused_adam", 1))
    for t in (1, 2):
        rt.step(ref, t)
        rt.step(off, t)
        torch.cuda.synchronize()
        rt.poll(ref)
        rt.poll(off)
        for r in ref:
            for k in ("master", "m", "v"):
                a = ref[r].tensors[k].view(torch.int32)
                b = off[r].tensors[k].view(torch.int32)
                assert torch.equal(a, b), (t, r, k)
            assert torch.equal(ref[r].tensors["shard"].view(torch.int16), off[r].tensors["shard"].view(torch.int16))
