"""Fused all-gather -> GEMM (SURVEY §8 f-4, P:349 / P:467): with option
"fused_ag" a gather pushes its shards chunk by chunk (ag_push_chunked_kernel)
and posts a value per landed chunk; the layer GEMMs that read the gathered
weights as their B operand do not wait for the whole gather on the compute
stream — the GEMM's TMA producer waits, per tile, for just the chunks its
loads cover.

Checked with N virtual ranks on one GPU (every rank's GEMM capped to 1/N of the
SMs so a GEMM waiting for another rank's chunks cannot keep that rank's GEMMs
off the device):
  * planned steps (prefetch + unshard and the plain S_0 schedule), Llama- and
    Mixtral-shaped layers, against the oracle (tests/oracle_check.py: loss,
    gradients element-wise, update bit-exact), with every push delayed 2 ms
    after its ready wait (option ag_delay_us) and released arena intervals
    poisoned to NaN (DC_DEBUG_POISON): a GEMM that read a chunk before it
    landed would read stale / NaN rows and fail the comparison;
  * the waits really moved into the GEMMs: under S_0 (each gather issued right
    before its consumer) with a 30 ms push delay, the profiled qkv op lasts
    >= 15 ms in fused mode (the GEMM starts and waits inside) and < 15 ms
    without (the compute stream waits before the op's start event).
"""
import json

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
PS = dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD


def _ranks(cfg, world, fused, delay_us):
    table = synth.param_table(cfg)
    ranks = rt.create_ranks(table, world, lr=LR, extra_flags=dc.DC_DEBUG_POISON)
    for st in ranks.values():
        dc.check(dc.lib.dc_set_option(st.ctx, b"fused_ag", int(fused)), st.ctx)
        dc.check(dc.lib.dc_set_option(st.ctx, b"ag_delay_us", delay_us), st.ctx)
    xs, ts = {}, {}
    for r in ranks:
        x, t = ost.rank_batch(cfg, r)
        xs[r], ts[r] = bf16_tensor(x), bf16_tensor(t)
    rt.attach_model(ranks, cfg, xs, ts)
    return table, ranks


@pytest.mark.parametrize("world,moe,passes", [(2, False, PS), (4, False, PS), (2, True, PS),
                                              (2, False, dc.DC_PASS_SHARD)])
def test_fused_ag_gemm_matches_oracle(world, moe, passes):
    cfg = synth.small_mixtral(layers=2, seq=128) if moe else synth.small_llama(layers=2, seq=128)
    table, ranks = _ranks(cfg, world, True, 2000)
    prof = rt.profile_json(ranks[0], tc=TC)
    sched = dc.plan(json.dumps(prof), 1 << 40, M_prefetch=1 << 22, passes=passes, strict=True)
    rt.bind(ranks, {r: sched for r in ranks})
    for s in (1, 2):
        check_step(ranks, table, cfg, world, s, LR, lambda: rt.step(ranks, s))


def _qkv_us(fused):
    cfg = synth.small_llama(layers=2, seq=128)
    _, ranks = _ranks(cfg, 2, fused, 30000)
    prof = rt.profile_json(ranks[0], tc=TC)
    sched = dc.plan(json.dumps(prof), 1 << 40, passes=dc.DC_PASS_SHARD)
    rt.bind(ranks, {r: sched for r in ranks})
    rt.step(ranks, 1)
    rt.step(ranks, 2, profile=True)
    torch.cuda.synchronize()
    rt.poll(ranks)
    p = json.loads(dc.model_profile_json(ranks[0].model))
    return [o["dur_us"] for o in p["ops"] if o["kind"] == "compute" and o.get("name") == "qkv"]


def test_fused_ag_waits_inside_the_gemm():
    fused, plain = _qkv_us(True), _qkv_us(False)
    assert fused and plain
    assert min(fused) >= 15000, fused
    assert max(plain) < 15000, plain


def test_fused_ag_option_rules():
    cfg = synth.small_llama(layers=1, seq=128)
    table = synth.param_table(cfg)
    ranks = rt.create_ranks(table, 2, lr=LR)
    st = ranks[0]
    assert dc.lib.dc_set_option(st.ctx, b"ag_delay_us", -1) == dc.DC_EINVAL
    xs = {r: bf16_tensor(ost.rank_batch(cfg, r)[0]) for r in ranks}
    rt.attach_model(ranks, cfg, xs, xs)
    sched = dc.plan(json.dumps(rt.profile_json(st, tc=TC)), 1 << 40, passes=dc.DC_PASS_SHARD)
    rt.bind(ranks, {r: sched for r in ranks})
    assert dc.lib.dc_set_option(st.ctx, b"fused_ag", 1) == dc.DC_ESTATE      # after the bind


@pytest.mark.parametrize("fused", [False, True])
def test_random_delay_injection_matches_oracle(fused):
    """SURVEY §5 race detection: every push, every release's ready posts and
    every reduce-scatter start after a random delay (option jitter_us, a
    counter-based hash of (seed, rank, op, step)), so the 4 virtual ranks
    interleave differently at every op; released arena intervals are poisoned.
    Two planned steps still match the oracle exactly."""
    cfg = synth.small_llama(layers=2, seq=128)
    table, ranks = _ranks(cfg, 4, fused, 0)
    for r, st in ranks.items():
        dc.check(dc.lib.dc_set_option(st.ctx, b"jitter_us", 3000), st.ctx)
        dc.check(dc.lib.dc_set_option(st.ctx, b"jitter_seed", 17 + r), st.ctx)
    prof = rt.profile_json(ranks[0], tc=TC)
    sched = dc.plan(json.dumps(prof), 1 << 40, M_prefetch=1 << 22, passes=PS, strict=True)
    rt.bind(ranks, {r: sched for r in ranks})
    for s in (1, 2):
        check_step(ranks, table, cfg, 4, s, LR, lambda: rt.step(ranks, s))
