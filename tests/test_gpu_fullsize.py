"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (CTA-pair tcgen05 GEMMs, rs_adam grid, planned schedule with prefetch +
selective unshard, strict), on outputs the oracle can compute one by one:

* layer outputs of sampled tokens: the synthetic layer is token-local (the
  attention core is the token-local surrogate, MoE routing depends only on the
  token index), so the oracle runs the layer on just those tokens, from the
  counter-generated weights and inputs (nothing taken from the GPU);
* the optimizer update of sampled shard elements: a property that holds at any
  size — the new fp32 master equals the oracle's fixed-order reduce-scatter
  (+0.0, ascending rank, x 1/N) and Adam step 1 applied to the generated
  initial value and the ranks' bf16 gradients left in the grad slots, bit for
  bit, and the bf16 shard is its RNE rounding.

* the whole step at N = 1: the oracle's fp64 sharded step of the 2-layer
  stack at T = 4096 (all host cores for its BLAS), compared like every small
  planned step (tests/oracle_check.py): loss, EVERY weight gradient element-wise
  (so the backward GEMMs with their grouped tile order and stream-K tails at
  K = 4096 / 14336 are checked at full size), the update bit-exact.

Llama-3-8B-shaped layers (h 4096, f 14336, 32/8 heads) at seq 2048, b = 2
(T = 4096) at N = 1 and N = 2 (virtual ranks); a Mixtral-8x7B-shaped layer at
T = 4096.  Tolerances: bf16 layer outputs and grads element-wise
(gpu_util.assert_bf16_close); update bit-exact.
"""
import ctypes as C
import dataclasses
import json

import numpy as np
import pytest
import torch

import synth
from oracle import model as om
from oracle import numerics as nx
from tests.gpu_util import assert_bf16_close, bf16_tensor, to_np
from tests.oracle_check import check_step

pytestmark = pytest.mark.gpu

dc = pytest.importorskip("paper_2504_09983_b200.dc")
from paper_2504_09983_b200 import runtime as rt  # noqa: E402

LR = 1e-3
PS = dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD


def _weights(table, layer, skip=()):
    """bf16-valued full weights of one layer from the generator (oracle side)."""
    W = {}
    for p in table:
        if p.layer != layer:
            continue
        if p.name in skip:
            continue
        v = np.ones(p.numel, np.float32) if p.k == 0.0 else synth.values(synth.SEED_WEIGHTS, p.id, 0, p.numel, p.k)
        W[p.name] = nx.rne_bf16(v).reshape(p.shape)
    return W


def _rows(seed, tokens, H):
    return np.stack([nx.rne_bf16(synth.values(seed, 0, t * H, H, synth.K_UNIT)) for t in tokens])


def _setup(cfg, world, step=True):
    table = synth.param_table(cfg)
    ranks = rt.create_ranks(table, world, lr=LR)
    xs, ts = {}, {}
    n = cfg.tokens * cfg.hidden
    for r in ranks:
        xs[r] = bf16_tensor(synth.values(synth.seed_inputs(r), 0, 0, n, synth.K_UNIT))
        ts[r] = bf16_tensor(synth.values(synth.seed_targets(r), 0, 0, n, synth.K_UNIT))
    rt.attach_model(ranks, cfg, xs, ts)
    frags = rt.offload_fragments(ranks[0], 256 << 20)
    prof = rt.profile_json(ranks[0], tc=[[4096, 20], [1 << 20, 40], [1 << 30, 2000]], frags=frags)
    total = torch.cuda.get_device_properties(0).total_memory
    sched = dc.plan(json.dumps(prof), int(0.9 * (total - 7 * (1 << 30))), passes=PS, strict=True)
    rt.bind(ranks, {r: sched for r in ranks})
    if step:
        rt.step(ranks, 1)
        torch.cuda.synchronize()
        rt.poll(ranks)
    return table, ranks


def _layer_out(st, layer, cfg):
    p = C.c_void_p()
    dc.check(dc.lib.dc_model_act_ptr(st.model, layer, 7, C.byref(p)))
    return rt.view(p.value, cfg.tokens * cfg.hidden, torch.bfloat16).view(cfg.tokens, cfg.hidden)


def _check_tokens(st, cfg, table, tokens, rank=0, skip=(), W=None):
    W = W if W is not None else _weights(table, 0, skip)
    x = _rows(synth.seed_inputs(rank), tokens, cfg.hidden)
    sub = dataclasses.replace(cfg, seq=len(tokens), batch=1)
    fwd = om.moe_layer_fwd if cfg.n_experts else om.llama_layer_fwd
    y_ref, _ = fwd(x, W, sub, nx.rne_bf16)
    y = to_np(_layer_out(st, 0, cfg)[torch.tensor(tokens, device="cuda")])
    return assert_bf16_close(y, y_ref, "sampled tokens %s" % tokens, rows=len(tokens))


def _check_update(ranks, table, world, n_sample=4096, seed=7):
    """Sampled elements of every param: master_new == Adam_1(init, RS(bf16 grads))."""
    rng = np.random.default_rng(seed)
    checked = 0
    slots = {}
    for r, st in ranks.items():
        for layer in (0, 1):
            s = C.c_void_p()
            dc.check(dc.lib.dc_grad_slot(st.ctx, layer, C.byref(s)), st.ctx)
            slots[(r, layer)] = s.value
    for r, st in ranks.items():
        master = st.tensors["master"]
        shard = st.tensors["shard"]
        for i, p in enumerate(table):
            if p.layer > 1:
                continue
            off, S = rt.shard_range(st, i)
            idx = np.unique(rng.integers(0, S, size=min(n_sample, S)))
            gi = torch.tensor(idx, device="cuda")
            goff = rt.grad_offset(st, i)
            # bf16 grads of element r*S + idx on every rank (padded full tensor in each slot)
            g = [to_np(rt.view(slots[(q, p.layer)] + goff, world * S, torch.bfloat16)[r * S + gi]).astype(np.float32)
                 for q in range(world)]
            full_idx = r * S + idx
            valid = full_idx < p.numel
            init = np.array([(1.0 if p.k == 0.0 else synth.values(synth.SEED_WEIGHTS, p.id, int(j), 1, p.k)[0])
                             if v else 0.0 for j, v in zip(full_idx, valid)], np.float32)   # zero padding
            gsum = nx.reduce_scatter([gq.reshape(-1) for gq in g], 1, 0) if world == 1 else None
            acc = np.zeros(len(idx), np.float32)
            for q in range(world):                     # +0.0, ascending rank, fp32
                acc = (acc + g[q]).astype(np.float32)
            if world == 1:
                assert np.array_equal(gsum, acc)
            gm = nx.scale_mean(acc, world)
            ref, _, _ = nx.adam_update(init, np.zeros_like(init), np.zeros_like(init), gm, 1, LR)
            got = master[off + gi].cpu().numpy()
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (r, p.name)
            sh = shard[off + gi].view(torch.int16).cpu().numpy().view(np.uint16)
            assert np.array_equal(sh, nx.bf16_bits(ref)), (r, p.name)
            checked += len(idx)
    return checked


def test_llama8b_fullsize_n1():
    cfg = dataclasses.replace(synth.LLAMA3_8B, layers=2, seq=2048, batch=2)
    table, ranks = _setup(cfg, 1)
    tokens = [0, 1, 255, 256, 1023, 2048, 3071, 4095]
    _check_tokens(ranks[0], cfg, table, tokens)
    assert _check_update(ranks, table, 1) > 9 * 2 * 1000


def test_llama8b_fullsize_n1_whole_step_vs_oracle():
    cfg = dataclasses.replace(synth.LLAMA3_8B, layers=2, seq=2048, batch=2)
    table, ranks = _setup(cfg, 1, step=False)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=len(__import__("os").sched_getaffinity(0))):
        check_step(ranks, table, cfg, 1, 1, LR, lambda: rt.step(ranks, 1))


def test_llama8b_fullsize_n2_virtual_ranks():
    """Two ranks: every layer weight is all-gathered by ag_push (or kept by the
    unshard pass) before use, so rank 1's sampled outputs check the gathers at
    full size; the update checks the reduce-scatter (rank order, 1/2)."""
    cfg = dataclasses.replace(synth.LLAMA3_8B, layers=2, seq=2048, batch=2)
    table, ranks = _setup(cfg, 2)
    W = _weights(table, 0)
    for r in (0, 1):
        _check_tokens(ranks[r], cfg, table, [3, 700, 2047, 4094], rank=r, W=W)
    assert _check_update(ranks, table, 2, n_sample=2048) > 9 * 2 * 2 * 500


def test_mixtral_fullsize_n1():
    """One Mixtral-8x7B-shaped layer at T = 4096 (E = 8 experts of f 14336,
    R = 1024 rows each).  Token pairs (8k, 8k+1) are routed to experts 0-2 both
    in the full batch and in a 2-token oracle batch, so only those experts'
    weights are generated (the others get empty stand-ins)."""
    cfg = dataclasses.replace(synth.MIXTRAL_8X7B, layers=1, seq=2048, batch=2)
    table, ranks = _setup_mixtral(cfg)
    skip = tuple("w%d_%d" % (j, e) for e in range(3, 8) for j in (1, 3, 2))
    W = _weights(table, 0, skip)
    H = cfg.hidden
    for e in range(3, 8):
        W["w1_%d" % e] = W["w3_%d" % e] = np.zeros((0, H))
        W["w2_%d" % e] = np.zeros((H, 0))
    for k in (0, 37, 511):
        _check_tokens(ranks[0], cfg, table, [8 * k, 8 * k + 1], W=W)


def _setup_mixtral(cfg):
    table = synth.param_table(cfg)
    ranks = rt.create_ranks(table, 1, lr=LR)
    n = cfg.tokens * cfg.hidden
    xs = {0: bf16_tensor(synth.values(synth.seed_inputs(0), 0, 0, n, synth.K_UNIT))}
    ts = {0: bf16_tensor(synth.values(synth.seed_targets(0), 0, 0, n, synth.K_UNIT))}
    rt.attach_model(ranks, cfg, xs, ts)
    prof = rt.profile_json(ranks[0])
    rt.bind(ranks, {0: dc.plan(json.dumps(prof), 1 << 50, passes=PS, strict=True)})
    rt.step(ranks, 1)
    torch.cuda.synchronize()
    rt.poll(ranks)
    return table, ranks
