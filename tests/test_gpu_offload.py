"""Adaptive offload (§4.4, Algorithm 2 + reload rule) on the
GPU path, with DC_DEBUG_POISON: once a fragment's D2H copy is synced the
device slice is overwritten with NaNs, so a missing or misordered reload
corrupts the Adam update.  Every offloaded step is checked against the
oracle's step from the GPU's states (tests/oracle_check.py) and must be
bit-identical to the same step without offload."""
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
        check_step(off, table, cfg, world, t, LR, lambda: rt.step(off, t))
        rt.poll(ref)
        for r in ref:
            for k in ("master", "m", "v"):
                a = ref[r].tensors[k].view(torch.int32)
                b = off[r].tensors[k].view(torch.int32)
                assert torch.equal(a, b), (t, r, k)
            assert torch.equal(ref[r].tensors["shard"].view(torch.int16), off[r].tensors["shard"].view(torch.int16))


@pytest.mark.parametrize("world,moe", [(1, False), (2, False), (1, True)])
def test_host_resident_states_bitexact_vs_resident(world, moe):
    """Reading D28 (host-resident offload): the offloaded (layer, m|v)
    fragments have no device array at all — each is reloaded into a ring slot
    of a small pool, updated there and written back right after its layer's
    update.  Three steps bit-identical to the all-resident step; the device m /
    v arrays shrink by the offloaded prefix and the pool is smaller than what
    it stands in for."""
    cfg = synth.small_mixtral(layers=3, seq=128) if moe else synth.small_llama(layers=3, seq=128)
    table = synth.param_table(cfg)
    n = sum(-(-p.numel // (8 * world)) * 8 for p in table)

    def make(defer):
        ranks = rt.create_ranks(table, world, lr=LR, host_pinned_bytes=8 * n + 4096, defer_states=defer)
        xs, ts = {}, {}
        for r in ranks:
            x, t = ost.rank_batch(cfg, r)
            xs[r], ts[r] = bf16_tensor(x), bf16_tensor(t)
        rt.attach_model(ranks, cfg, xs, ts)
        return ranks

    ref = make(False)
    prof = rt.profile_json(ref[0])
    rt.bind(ref, {r: dc.plan(json.dumps(prof), 1 << 40, passes=dc.DC_PASS_SHARD) for r in ref})
    off = make(True)
    for st in off.values():
        frags = rt.offload_fragments(st, rt.layer_state_bytes(table, world))
    assert len(frags) == 2 * cfg.layers                       # one per (layer, state)
    prof = rt.profile_json(off[0], frags=frags)
    peak = max(o["p_mem"] + o["transient"] for o in prof["ops"])
    m_opt = sum(f["bytes"] for f in frags)
    # the host-state reload rule (D28) for the Llama cases, the paper's for MoE
    sched = dc.plan(json.dumps(prof), peak + m_opt - frags[0]["bytes"] - frags[1]["bytes"] - frags[2]["bytes"],
                    passes=dc.DC_PASS_SHARD | dc.DC_PASS_OFFLOAD | (0 if moe else dc.DC_PASS_HOST_STATES),
                    strict=True)
    plan = json.loads(dc.schedule_json(sched))
    assert plan["offload"] == [0, 1, 2]                       # layer 0 m, v and layer 1 m
    rt.bind(off, {r: sched for r in off})
    # MoE case: pinned slots sized from the plan; N=2: two extra ring slots (round-robin reuse)
    info = rt.bind_host_states(off, alloc_host=moe, extra_slots=2 if world == 2 else 0)
    E = off[0].layout.shard_elems
    for r, (mf, vf, pool, hb) in info.items():
        assert hb == sum(frags[i]["bytes"] for i in plan["offload"])
        assert mf > vf > 0                                     # m: layers 0-1 offloaded, v: layer 0
        assert off[r].tensors["m"].numel() == E - mf and off[r].tensors["v"].numel() == E - vf
        assert 0 < pool <= sum(frags[i]["bytes"] for i in plan["offload"]) + (2 * frags[0]["bytes"] if world == 2 else 0)
    # a DC_WRITEBACK outside host-state mode is refused
    rt.offload_fragments(ref[0], rt.layer_state_bytes(table, world))
    assert dc.lib.dc_offload(ref[0].ctx, 0, dc.DC_WRITEBACK, ref[0].streams[3].cuda_stream) == dc.DC_ESTATE
    for t in (1, 2, 3):
        rt.step(ref, t)
        check_step(off, table, cfg, world, t, LR, lambda: rt.step(off, t))
        rt.poll(ref)
        for r in ref:
            for k in ("master", "shard"):
                dt = torch.int16 if k == "shard" else torch.int32
                assert torch.equal(ref[r].tensors[k].view(dt), off[r].tensors[k].view(dt)), (t, r, k)
            m_ref, v_ref = ref[r].tensors["m"].cpu(), ref[r].tensors["v"].cpu()
            m_off, v_off = rt.full_states(off[r])
            assert torch.equal(m_ref.view(torch.int32), m_off.view(torch.int32)), (t, r, "m")
            assert torch.equal(v_ref.view(torch.int32), v_off.view(torch.int32)), (t, r, "v")


def test_offload_all_sync_baseline_bitexact():
    """The paper's comparison point for adaptive offload (option
    offload_all_sync): no optimizer state on the device, every fragment
    reloaded synchronously before its layer's update and written back after;
    bit-identical to the all-resident step."""
    cfg = synth.small_llama(layers=3, seq=128)
    table = synth.param_table(cfg)
    n = sum(-(-p.numel // 8) * 8 for p in table)
    runs = []
    for sync in (False, True):
        ranks = rt.create_ranks(table, 1, lr=LR, host_pinned_bytes=8 * n + 4096, defer_states=sync)
        x, t = ost.rank_batch(cfg, 0)
        rt.attach_model(ranks, cfg, {0: bf16_tensor(x)}, {0: bf16_tensor(t)})
        st = ranks[0]
        frags = rt.offload_fragments(st, rt.layer_state_bytes(table, 1))
        prof = rt.profile_json(st, frags=frags)
        rt.bind(ranks, {0: dc.plan(json.dumps(prof), 1 << 40, passes=dc.DC_PASS_SHARD)})
        if sync:
            dc.check(dc.lib.dc_model_set_option(st.model, b"offload_all_sync", 1))
            mf, vf, pool, hb = rt.bind_host_states(ranks)[0]
            assert mf == vf == st.layout.shard_elems and pool > 0 and hb == 8 * st.layout.shard_elems
            assert dc.lib.dc_model_set_option(st.model, b"offload_all_sync", 0) == dc.DC_ESTATE
        for s in (1, 2, 3):
            if sync:    # the paper's baseline against the oracle itself
                check_step(ranks, table, cfg, 1, s, LR, lambda: rt.step(ranks, s))
            else:
                rt.step(ranks, s)
                torch.cuda.synchronize()
                rt.poll(ranks)
        runs.append(st)
    a, b = runs
    for k in ("master", "shard"):
        dt = torch.int16 if k == "shard" else torch.int32
        assert torch.equal(a.tensors[k].view(dt), b.tensors[k].view(dt)), k
    m_b, v_b = rt.full_states(b)
    assert torch.equal(a.tensors["m"].cpu().view(torch.int32), m_b.view(torch.int32))
    assert torch.equal(a.tensors["v"].cpu().view(torch.int32), v_b.view(torch.int32))
