"""One GPU training step checked directly against the oracle (no GPU-vs-GPU
comparison): used by every -m gpu test of a planned step (plain, prefetch /
unshard, offload and host-resident states, activation checkpointing,
copy-engine gathers, CUDA-graph replay, gradient accumulation, MoE layers).

The oracle step starts from the GPU's own states before the step (fp32 master /
m / v and the bf16 shard), so every step of a multi-step run is checked, not
only the first:
  * loss of every rank and micro-step within 2e-2 (BASELINE north star);
  * the bf16 gradients left in the grad slots (the last two layers of the
    backward) element-wise against the oracle's gradients
    (gpu_util.assert_bf16_close);
  * the update bit-exact: master / m / v / shard == the oracle's
    reduce-scatter + 1/(N n) + Adam (oracle.numerics.rs_adam_shard) of the
    ranks' own bf16 gradients (and, with accumulation, the GPU's fp32
    accumulator of the earlier micro-steps, itself checked against the
    oracle's);
  * params whose gradients are no longer in a slot (layers >= 2): master
    within 2.02 lr of the oracle's update (Adam moves an element by at most
    ~lr per step, so a missed or doubled update fails).
"""
import numpy as np
import torch

from oracle import numerics as nx
from oracle import step as ost
from tests.gpu_util import assert_bf16_close, slot_grads

F32 = np.float32


def _host_states(st):
    from paper_2504_09983_b200 import runtime as rt
    return rt.full_states(st)


def snapshot(ranks, table):
    """Per rank and param: fp32 master, m, v and the bf16 shard bits (numpy)."""
    from paper_2504_09983_b200 import runtime as rt
    out = {}
    for r, st in ranks.items():
        m_all, v_all = (x.numpy() for x in _host_states(st))
        ms = st.tensors["master"].cpu().numpy()
        sh = st.tensors["shard"].view(torch.int16).cpu().numpy().view(np.uint16)
        acc = st.tensors["acc"].cpu().numpy() if "acc" in st.tensors else None
        per = []
        for i in range(len(table)):
            off, n = rt.shard_range(st, i)
            per.append(dict(master=ms[off:off + n].copy(), m=m_all[off:off + n].copy(),
                            v=v_all[off:off + n].copy(), shard=sh[off:off + n].copy(),
                            acc=None if acc is None else acc[off:off + n].copy()))
        out[r] = per
    return out


def oracle_from(snap, table, world, step_before):
    """An oracle ShardedState holding exactly the GPU's states."""
    o = ost.ShardedState(table, world, bf16=True)
    for r in range(world):
        for i in range(len(table)):
            s = snap[r][i]
            o.master[r][i] = s["master"].astype(F32)
            o.m[r][i] = s["m"].astype(F32)
            o.v[r][i] = s["v"].astype(F32)
            o.shard[r][i] = nx.bf16_to_f32(s["shard"])
    o.t = step_before
    return o


def check_step(ranks, table, cfg, world, step_t, lr, run_step, micro_steps=1, loss_rel=2e-2, skip_grads=()):
    """Snapshot, run the GPU step (`run_step()`), run the oracle step from the
    snapshot, compare.  Returns the oracle's losses."""
    from paper_2504_09983_b200 import runtime as rt
    before = snapshot(ranks, table)
    run_step()
    torch.cuda.synchronize()
    rt.poll(ranks)
    oracle = oracle_from(before, table, world, step_t - 1)
    o_losses, o_grads = ost.sharded_step(oracle, cfg, lr=lr, micro_steps=micro_steps)
    after = snapshot(ranks, table)
    L = max(p.layer for p in table) + 1
    slot_layers = {0, 1} if L >= 2 else {0}
    for r, st in ranks.items():
        got = rt.view(rt.loss_ptr(st), micro_steps, torch.float32).cpu().numpy()
        for mu in range(micro_steps):
            ref = oracle.micro_losses[mu][r]
            assert abs(got[mu] - ref) <= loss_rel * abs(ref), ("loss", r, mu, got[mu], ref)
    grads = {r: slot_grads(st, table, world, layers=slot_layers) for r, st in ranks.items()}
    for r in ranks:
        for i, p in enumerate(table):
            if p.layer not in slot_layers or i in skip_grads:
                continue
            g = grads[r][i]
            assert_bf16_close(g[:p.numel], o_grads[r][i][:p.numel], "grad r%d %s" % (r, p.name),
                              rows=p.shape[0] if len(p.shape) == 2 else None)
            assert not g[p.numel:].any(), ("padding", r, p.name)
    for r in ranks:
        for i, p in enumerate(table):
            b, a = before[r][i], after[r][i]
            if p.layer in slot_layers and i not in skip_grads:
                acc = None
                if micro_steps > 1:
                    acc = a["acc"]          # FINAL mode reads the accumulator, leaves it as acc_{n-2}
                    assert_bf16_close(acc, oracle.acc[r][i], "grad accumulator r%d %s" % (r, p.name), ulps=8)
                e_mst, e_m, e_v, e_sh = nx.rs_adam_shard([grads[q][i] for q in range(world)], b["master"], b["m"],
                                                         b["v"], world, r, step_t, lr, acc=acc,
                                                         micro_steps=micro_steps)
                for k, e in (("master", e_mst), ("m", e_m), ("v", e_v)):
                    assert a[k].tobytes() == np.asarray(e, F32).tobytes(), ("update", r, p.name, k)
                assert np.array_equal(a["shard"], nx.bf16_bits(e_sh)), ("update", r, p.name, "shard")
            else:
                d = np.abs(a["master"].astype(np.float64) - oracle.master[r][i])
                assert d.max() <= 2.02 * lr, ("master", r, p.name, d.max())
                assert np.array_equal(a["shard"], nx.bf16_bits(nx.rne_bf16(a["master"]))), ("shard", r, p.name)
    return o_losses
