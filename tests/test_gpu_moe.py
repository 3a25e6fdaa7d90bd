"""Mixtral-shaped MoE layers (PAPER.md line 440:
Mixtral 8x7B) through the sharded step on the GPU, against the oracle's
moe_layer_fwd/bwd (oracle/model.py) and its N-rank simulated sharded step.

31 tensors per layer at E = 8 (many medium shards: the small-message gather
regime of P:471).  Tolerances as for the Llama-shaped stack (BASELINE north
star), checked against the oracle's step from the GPU's states
(tests/oracle_check.py): loss within 2e-2, bf16 layer outputs and grads
element-wise, the update bit-exact as the oracle's reduce-scatter + Adam of the
ranks' bf16 grads.
"""
import ctypes as C
import json

import numpy as np
import pytest
import torch

import synth
from oracle import model as om
from oracle import numerics as nx
from oracle import step as ost
from tests.gpu_util import assert_bf16_close, bf16_tensor, to_np
from tests.oracle_check import check_step

pytestmark = pytest.mark.gpu

dc = pytest.importorskip("paper_2504_09983_b200.dc")
from paper_2504_09983_b200 import runtime as rt  # noqa: E402

LR = 1e-3
PS = dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD


def _setup(cfg, world, passes, checkpoint=False, M=1 << 40, prefetch=1 << 22):
    table = synth.param_table(cfg)
    ranks = rt.create_ranks(table, world, lr=LR)
    xs, ts = {}, {}
    for r in ranks:
        x, t = ost.rank_batch(cfg, r)
        xs[r], ts[r] = bf16_tensor(x), bf16_tensor(t)
    rt.attach_model(ranks, cfg, xs, ts, checkpoint=checkpoint)
    prof = rt.profile_json(ranks[0], tc=[[4096, 10], [1 << 20, 20], [1 << 26, 400]])
    sched = dc.plan(json.dumps(prof), M, M_prefetch=prefetch, passes=passes, strict=True)
    rt.bind(ranks, {r: sched for r in ranks})
    return table, ranks, prof


def _loss(st):
    return rt.view(rt.loss_ptr(st), 1, torch.float32).item()


def test_moe_s0_matches_workload_graph():
    """The executor's compute ops (profile skeleton) are synth's MoE op graph,
    in order, with the same consumed params; gathers/releases follow S_0."""
    cfg = synth.small_mixtral(layers=2, seq=128)
    for ck in (False, True):
        _, ranks, prof = _setup(cfg, 1, dc.DC_PASS_SHARD, checkpoint=ck)
        got = [(o["name"], o["phase"], o["layer"], o["params"]) for o in prof["ops"] if o["kind"] in ("compute", "rs")]
        want = [(o["name"], o["phase"], o["layer"], o["params"]) for o in synth.compute_ops(cfg, checkpoint=ck)]
        assert got == want
        n_ag = sum(o["kind"] == "ag" for o in prof["ops"])
        assert n_ag == 2 * len(synth.param_table(cfg))        # one per param per phase (S_0)


@pytest.mark.parametrize("world,passes", [(1, dc.DC_PASS_SHARD), (2, PS), (4, PS)])
def test_moe_step_matches_oracle(world, passes):
    cfg = synth.small_mixtral(layers=2, seq=128)
    table, ranks, _ = _setup(cfg, world, passes)
    for t in (1, 2):
        check_step(ranks, table, cfg, world, t, LR, lambda: rt.step(ranks, t))


def test_moe_layer_outputs_gates_and_routing():
    """Per layer, given the layer's own input on the GPU (the bf16 x for layer 0,
    the GPU's layer-0 output for layer 1): the gates (fp32), the expert-major
    token gather X (exact: a permutation of h2) and the layer output y against
    the oracle's layer on that input.  (Whole-stack chains against the oracle's
    own activations: test_moe_step_matches_oracle.)"""
    cfg = synth.small_mixtral(layers=2, seq=128)
    table, ranks, _ = _setup(cfg, 1, dc.DC_PASS_SHARD)
    st = ranks[0]
    ref = ost.ShardedState(table, 1, bf16=True)
    full = ref.gathered(0)
    P = len(table) // cfg.layers
    Ws = [{p.name: full[l * P + j].reshape(p.shape) for j, p in enumerate(table[l * P:(l + 1) * P])}
          for l in range(cfg.layers)]
    x, t = ost.rank_batch(cfg, 0)
    h = nx.rne_bf16(x)
    rt.step(ranks, 1)
    torch.cuda.synchronize()
    T, H, E = cfg.tokens, cfg.hidden, cfg.n_experts

    def act(l, which, n, dt):
        p = C.c_void_p()
        dc.check(dc.lib.dc_model_act_ptr(st.model, l, which, C.byref(p)))
        return to_np(rt.view(p.value, n, dt))

    for l in range(cfg.layers):
        y_ref, c = om.moe_layer_fwd(h, Ws[l], cfg, nx.rne_bf16)
        g01 = act(l, 10, 2 * T, torch.float32).reshape(T, 2)
        for k in (0, 1):    # fp32 gates (softmax of two bf16-input fp32 logits)
            ref = np.asarray(c["g%d" % k], np.float64)
            assert np.all(np.abs(g01[:, k] - ref) <= 1e-3 * np.abs(ref) + 1e-6), ("gate", l, k)
        assert np.all(np.abs(g01.sum(axis=1) - 1.0) <= 1e-6)
        h2 = act(l, 4, T * H, torch.bfloat16).reshape(T, H)
        X = act(l, 11, 2 * T * H, torch.bfloat16).reshape(E, 2 * T // E, H)
        for e in range(E):
            assert np.array_equal(X[e], h2[om.expert_tokens(T, E, e)])
        y = act(l, 7, T * H, torch.bfloat16).reshape(T, H)
        assert_bf16_close(y, y_ref, "moe layer %d output" % l, rows=T)
        h = y


@pytest.mark.parametrize("world,passes", [(1, dc.DC_PASS_SHARD), (2, PS)])
def test_moe_checkpointing_bitexact(world, passes):
    """Layer activation checkpointing on MoE layers: recompute re-runs the
    router, gather and every expert's forward from the saved layer input;
    both steps checked against the oracle, and bit-identical states and loss to
    the non-recomputing steps."""
    cfg = synth.small_mixtral(layers=2, seq=128)
    runs = {}
    for ck in (False, True):
        table, ranks, _ = _setup(cfg, world, passes, checkpoint=ck)
        for t in (1, 2):
            if ck:      # the recomputing step against the oracle itself
                check_step(ranks, table, cfg, world, t, LR, lambda: rt.step(ranks, t))
            else:
                rt.step(ranks, t)
                torch.cuda.synchronize()
                rt.poll(ranks)
        runs[ck] = ranks
    a, b = runs[False], runs[True]
    assert b[0].tensors["act"].numel() < a[0].tensors["act"].numel()
    for r in a:
        for k in ("master", "m", "v", "shard"):
            x, y = a[r].tensors[k], b[r].tensors[k]
            assert torch.equal(x.view(torch.int16) if k == "shard" else x.view(torch.int32),
                               y.view(torch.int16) if k == "shard" else y.view(torch.int32)), (r, k)
        assert _loss(a[r]) == _loss(b[r])


def test_moe_options_and_shape_errors():
    cfg = synth.small_mixtral(layers=1, seq=128)
    _, ranks, _ = _setup(cfg, 1, dc.DC_PASS_SHARD)
    st = ranks[0]
    assert dc.lib.dc_model_set_option(st.model, b"fused_adam", 1) == dc.DC_EINVAL
    assert dc.lib.dc_model_set_option(st.model, b"side_adam", 1) == dc.DC_EINVAL
    # a Llama-shaped model on a MoE param table is refused
    d = dc.ModelDims(cfg.hidden, cfg.ffn, cfg.n_heads, cfg.n_kv, cfg.head_dim, cfg.layers, cfg.tokens, 0, 0)
    m = C.c_void_p()
    assert dc.lib.dc_model_create(st.ctx, C.byref(d), C.byref(m)) == dc.DC_EINVAL
    # tokens must split evenly into 2T/E rows per expert with R % 8 == 0
    d = dc.ModelDims(cfg.hidden, cfg.ffn, cfg.n_heads, cfg.n_kv, cfg.head_dim, cfg.layers, 136, 0, 8)
    assert dc.lib.dc_model_create(st.ctx, C.byref(d), C.byref(m)) == dc.DC_EINVAL
