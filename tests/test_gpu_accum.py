"""Gradient accumulation (§4.3, §5 lines
474-478): n micro-steps per optimizer step, each reduce-scattered into the
partitioned fp32 accumulator, Adam once on (acc + rs) / (N n).  The planned
schedule (selective unshard keeps parameters gathered across micro-steps)
runs through dc_model_step; results vs the oracle's accumulated sharded step.

Every step is checked against the oracle's accumulated step from the GPU's
states (tests/oracle_check.py): losses of every micro-step, element-wise
grads and fp32 accumulator, and the update bit-exact."""
import json

import numpy as np
import pytest
import torch

import synth
from oracle import step as ost
from tests.gpu_util import bf16_tensor
from tests.oracle_check import check_step

pytestmark = pytest.mark.gpu

dc = pytest.importorskip("paper_2504_09983_b200.dc")
from paper_2504_09983_b200 import runtime as rt  # noqa: E402

LR = 1e-3
TC = [[4096, 10], [1 << 20, 20], [1 << 26, 400]]


def _batches(cfg, r, n, duplicate=False):
    xs, ts = zip(*[ost.rank_batch(cfg, r, 0 if duplicate else mu) for mu in range(n)])
    return bf16_tensor(np.stack(xs)), bf16_tensor(np.stack(ts))


def _ranks(cfg, world, n, duplicate=False, **kw):
    table = synth.llama_param_table(cfg)
    ranks = rt.create_ranks(table, world, lr=LR, micro_steps=n, **kw)
    xs, ts = {}, {}
    for r in ranks:
        xs[r], ts[r] = _batches(cfg, r, n, duplicate)
    rt.attach_model(ranks, cfg, xs, ts)
    return table, ranks


def _plan_bind(ranks, passes, M=1 << 40, frags=None):
    prof = rt.profile_json(ranks[0], tc=TC, frags=frags)
    sched = dc.plan(json.dumps(prof), M, M_prefetch=1 << 22, passes=passes, strict=True)
    rt.bind(ranks, {r: sched for r in ranks})
    return prof, json.loads(dc.schedule_json(sched))


def _state(st):
    return {k: st.tensors[k].view(torch.int16 if k == "shard" else torch.int32).clone()
            for k in ("master", "m", "v", "shard")}


@pytest.mark.parametrize("world,n,passes", [
    (1, 2, dc.DC_PASS_SHARD),
    (2, 2, dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD),
    (2, 3, dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH),
])
def test_accumulated_step_matches_oracle(world, n, passes):
    cfg = synth.small_llama(layers=2, seq=128)
    table, ranks = _ranks(cfg, world, n)
    prof, plan = _plan_bind(ranks, passes)
    assert sum(o["kind"] == "rs" for o in prof["ops"]) == n * cfg.layers
    if passes & dc.DC_PASS_UNSHARD:
        # unsharded params are gathered once for all n micro-steps
        n_ag0 = sum(o["kind"] == "ag" for o in prof["ops"])
        n_ag = sum(len(o.get("members", [0])) for o in plan["ops"] if o["kind"] == "ag")
        assert plan["unshard"] and n_ag < n_ag0
    for t in (1, 2):
        check_step(ranks, table, cfg, world, t, LR, lambda: rt.step(ranks, t), micro_steps=n)


@pytest.mark.parametrize("world", [1, 2])
def test_duplicated_micro_batches_equal_single_step(world):
    """n = 2 copies of the same micro-batch: acc + rs = 2 rs exactly and
    fp32(1/(2N)) = fp32(1/N) / 2 exactly, so the update is bit-identical to
    the n = 1 step on that micro-batch."""
    cfg = synth.small_llama(layers=2, seq=128)
    _, one = _ranks(cfg, world, 1)
    _, two = _ranks(cfg, world, 2, duplicate=True)
    passes = dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD
    _plan_bind(one, passes)
    _plan_bind(two, passes)
    for t in (1, 2):
        rt.step(one, t)
        rt.step(two, t)
        torch.cuda.synchronize()
        rt.poll(one)
        rt.poll(two)
        for r in one:
            a, b = _state(one[r]), _state(two[r])
            for k in a:
                assert torch.equal(a[k], b[k]), (t, r, k)
            l1 = rt.view(rt.loss_ptr(one[r]), 1, torch.float32).item()
            l2 = rt.view(rt.loss_ptr(two[r]), 2, torch.float32).tolist()
            assert l2 == [l1, l1]


def test_accumulated_offload_bitexact_vs_resident():
    """Adaptive offload with n = 2: the optimizer states leave during the first
    micro-step's forward and return before the last micro-step's final
    reduce-scatter; bit-identical to the resident run (with NaN poison)."""
    cfg = synth.small_llama(layers=2, seq=128)
    world, n = 2, 2
    table = synth.llama_param_table(cfg)
    nel = sum(-(-p.numel // (8 * world)) * 8 for p in table)
    _, ref = _ranks(cfg, world, n)
    _plan_bind(ref, dc.DC_PASS_SHARD)
    _, off = _ranks(cfg, world, n, host_pinned_bytes=8 * nel + 4096, extra_flags=dc.DC_DEBUG_POISON)
    frags = None
    for st in off.values():
        frags = rt.offload_fragments(st, 128 * 1024)
    prof = rt.profile_json(off[0], tc=TC, frags=frags)
    peak = max(o["p_mem"] + o["transient"] for o in prof["ops"])
    m_opt = sum(f["bytes"] for f in frags)
    _, plan = _plan_bind(off, dc.DC_PASS_SHARD | dc.DC_PASS_OFFLOAD, M=peak + m_opt // 2, frags=frags)
    assert plan["offload"]
    for t in (1, 2):
        rt.step(ref, t)
        check_step(off, table, cfg, world, t, LR, lambda: rt.step(off, t), micro_steps=n)
        rt.poll(ref)
        for r in ref:
            a, b = _state(ref[r]), _state(off[r])
            for k in a:
                assert torch.equal(a[k], b[k]), (t, r, k)
