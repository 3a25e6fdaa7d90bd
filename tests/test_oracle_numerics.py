"""Pins for oracle/numerics.py, oracle/model.py and oracle/step.py.

Each test ties the oracle to something other than itself: a library
(ml_dtypes / torch conversions, torch.optim.Adam, torch.autograd), a closed
form (Adam's first step), brute force in fp64, or an invariant the paper fixes
(the sharded step equals the unsharded step, §5.6)."""
import numpy as np
import pytest
import torch

import synth
from oracle import numerics as nx
from oracle import model as om
from oracle import step as ost

F32 = np.float32


# ---------------------------------------------------------------- bf16 RNE
def test_rne_bf16_matches_libraries():
    import ml_dtypes
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(F32),
                        (rng.standard_normal(1000) * 1e-30).astype(F32),
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 3.0e38], F32)])
    # exact ties: mantissa low half == 0x8000 -> round to even
    ties = (np.arange(1, 2000, dtype=np.uint32) << 16 | 0x8000).view(F32)
    x = np.concatenate([x, ties, -ties])
    mine = nx.bf16_bits(x)
    lib = x.astype(ml_dtypes.bfloat16).view(np.uint16)
    assert np.array_equal(mine, lib)
    tor = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(mine, tor)


# ---------------------------------------------------------------- shards / gather
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_gather_roundtrip(world):
    rng = np.random.default_rng(world)
    for numel in [1, 7, 8, 9, 63, 64, 65, 1000, 4096 * 3 + 5]:
        full = rng.standard_normal(numel).astype(F32)
        S = nx.shard_len(numel, world)
        assert S % 8 == 0 and S * world >= numel and (S - 8) * world < numel
        shards = [nx.shard_of(full, world, r) for r in range(world)]
        assert all(s.size == S for s in shards)
        back = nx.all_gather(shards, numel)
        assert back.tobytes() == full.tobytes()          # bit-exact
        pad = nx.all_gather_padded(shards)
        assert not pad[numel:].any()                      # zero padding


def test_reduce_scatter_vs_bruteforce():
    rng = np.random.default_rng(1)
    N, S = 8, 4096
    grads = [nx.rne_bf16(rng.standard_normal(N * S).astype(F32)) for _ in range(N)]
    for r in range(N):
        got = nx.reduce_scatter(grads, N, r)
        ref = np.sum(np.stack([g[r * S:(r + 1) * S].astype(np.float64) for g in grads]), axis=0)
        err = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3)
        assert err.max() <= 1e-6
    # small integers are summed exactly in fp32
    ints = [np.full(N * S, q + 1, F32) for q in range(N)]
    assert np.all(nx.reduce_scatter(ints, N, 3) == sum(range(1, N + 1)))
    # ascending order starting from +0.0: -0.0 inputs give +0.0
    negz = [np.full(N * S, -0.0, F32) for _ in range(N)]
    assert not np.signbit(nx.reduce_scatter(negz, N, 0)).any()


# ---------------------------------------------------------------- Adam
def test_adam_vs_torch_optim():
    """Per step, from torch's own pre-step state: <= 1 ulp-level differences
    (torch's vectorised CPU kernels may contract into FMA), >95% bit-equal."""
    rng = np.random.default_rng(2)
    n = 65536
    p0 = (rng.standard_normal(n) * 0.02).astype(F32)
    tp = torch.nn.Parameter(torch.from_numpy(p0.copy()))
    opt = torch.optim.Adam([tp], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, foreach=False)
    m, v = np.zeros(n, F32), np.zeros(n, F32)
    for t in range(1, 6):
        g = (rng.standard_normal(n) * 1e-2).astype(F32)
        p_before = tp.detach().numpy().copy()
        tp.grad = torch.from_numpy(g.copy())
        opt.step()
        p, m2, v2 = nx.adam_update(p_before, m, v, g, t, lr=1e-3)
        tm = opt.state[tp]["exp_avg"].numpy().copy()
        tv = opt.state[tp]["exp_avg_sq"].numpy().copy()
        tpn = tp.detach().numpy()
        assert np.max(np.abs(tm - m2)) <= 2e-9
        assert np.max(np.abs(tv - v2) / np.maximum(tv, 1e-12)) <= 1e-6
        assert np.max(np.abs(tpn - p)) <= 2 * np.max(np.spacing(np.abs(tpn)))
        assert np.mean(tpn == p) > 0.95
        m, v = tm, tv


def test_adam_first_step_closed_form():
    """t=1: m = 0.1 g, v = 0.001 g^2, s = 10 lr, c = sqrt(0.001), d = |g| + eps,
    so p1 = p0 - lr * g / (|g| + eps)."""
    rng = np.random.default_rng(3)
    g = (rng.standard_normal(10000) * 1e-3).astype(F32)
    p0 = (rng.standard_normal(10000) * 0.02).astype(F32)
    lr = 1e-3
    p1, m1, v1 = nx.adam_update(p0, np.zeros_like(g), np.zeros_like(g), g, 1, lr=lr)
    assert np.allclose(m1, 0.1 * g.astype(np.float64), rtol=2e-7, atol=0)
    assert np.allclose(v1, 0.001 * g.astype(np.float64) ** 2, rtol=5e-7, atol=0)
    expect = p0.astype(np.float64) - lr * g / (np.abs(g.astype(np.float64)) + 1e-8)
    # a few roundings of the lr-sized update, one of the result
    tol = 4 * np.spacing(np.float32(lr)) + np.spacing(np.abs(p1)).astype(np.float64)
    assert np.all(np.abs(p1 - expect) <= tol)


def test_adam_zero_padding_stays_zero():
    z = np.zeros(64, F32)
    p, m, v = z, z, z
    for t in range(1, 4):
        p, m, v = nx.adam_update(p, m, v, z, t)
    assert not p.any() and not m.any() and not v.any()
    assert not np.signbit(p).any()


# ---------------------------------------------------------------- MLP (config 1)
def _mlp_params():
    cfg = synth.MLP_CONFIG1
    table = synth.mlp_param_table(cfg)
    full = ost.init_full_params(table)
    return cfg, [(full[2 * l].reshape(256, 256), full[2 * l + 1]) for l in range(4)]


def test_mlp_fwd_bwd_vs_torch_autograd():
    cfg, params = _mlp_params()
    x, t = ost.rank_batch(cfg, 0)
    loss, grads = om.mlp_fwd_bwd(x, t, params)
    tw = [(torch.tensor(W, requires_grad=True), torch.tensor(b, requires_grad=True)) for W, b in params]
    h = torch.tensor(x)
    for l, (W, b) in enumerate(tw):
        h = h @ W.T + b
        if l < 3:
            h = torch.relu(h)
    tl = (0.5 * (h - torch.tensor(t)) ** 2).mean()
    tl.backward()
    assert abs(tl.item() - loss) <= 1e-6 * abs(loss)
    for (dW, db), (W, b) in zip(grads, tw):
        assert np.max(np.abs(dW - W.grad.numpy())) <= 1e-6 * np.max(np.abs(W.grad.numpy())) + 1e-12
        assert np.max(np.abs(db - b.grad.numpy())) <= 1e-6 * np.max(np.abs(b.grad.numpy())) + 1e-12


def test_mlp_sharded_equals_unsharded_bitexact():
    """The invariant of PAPER.md §5.6: fully-sharded == data-parallel, 3 steps."""
    cfg = synth.MLP_CONFIG1
    table = synth.mlp_param_table(cfg)
    N = 2
    sh = ost.ShardedState(table, N, bf16=False)
    rp = ost.ReplicatedState(table, N, bf16=False)
    for _ in range(3):
        l1, _ = ost.sharded_step(sh, cfg, lr=1e-3)
        l2 = ost.replicated_step(rp, cfg, lr=1e-3)
        assert l1 == l2
        for i, p in enumerate(table):
            got = nx.all_gather([sh.master[r][i] for r in range(N)], p.numel)
            assert got.tobytes() == rp.master[i].tobytes()
            gm = nx.all_gather([sh.m[r][i] for r in range(N)], p.numel)
            assert gm.tobytes() == rp.m[i].tobytes()


def test_mlp_sharded_vs_full_batch():
    """N ranks x b samples == one process with N*b samples, up to summation order."""
    cfg = synth.MLP_CONFIG1
    table = synth.mlp_param_table(cfg)
    N = 2
    full = ost.init_full_params(table)
    params = [(full[2 * l].reshape(256, 256), full[2 * l + 1]) for l in range(4)]
    xs, ts = zip(*[ost.rank_batch(cfg, r) for r in range(N)])
    _, g_full = om.mlp_fwd_bwd(np.concatenate(xs), np.concatenate(ts), params)
    sh = ost.ShardedState(table, N, bf16=False)
    _, gp = ost.sharded_step(sh, cfg, lr=1e-3)
    for i, p in enumerate(table):
        S = sh.S[i]
        red = np.concatenate([nx.scale_mean(nx.reduce_scatter([gp[q][i] for q in range(N)], N, r), N)
                              for r in range(N)])[:p.numel]
        ref = (g_full[i // 2][i % 2]).reshape(-1)
        assert np.max(np.abs(red - ref)) <= 1e-5 * np.max(np.abs(ref))


# ---------------------------------------------------------------- Llama-shaped layer
def _small_weights(cfg, seed=5):
    table = synth.llama_param_table(cfg)
    full = ost.init_full_params(table)
    P = 9
    Ws = []
    for l in range(cfg.layers):
        W = {}
        for j, p in enumerate(table[l * P:(l + 1) * P]):
            w = full[l * P + j].reshape(p.shape)
            if p.k == 0.0:   # perturb gains so their gradient path is exercised
                w = w + synth.values(seed, p.id, 0, p.numel, 0.2)
            W[p.name] = nx.rne_bf16(w)
        Ws.append(W)
    return Ws


def _torch_stack(x, t, Ws, cfg):
    x = torch.tensor(x, dtype=torch.float64)
    TW = [{k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in W.items()} for W in Ws]

    def rms(z, g):
        return z * torch.rsqrt((z * z).mean(1, keepdim=True) + om.RMS_EPS) * g

    grp = cfg.n_heads // cfg.n_kv
    h = x
    for W in TW:
        h1 = rms(h, W["attn_norm"])
        q, k, v = h1 @ W["wq"].T, h1 @ W["wk"].T, h1 @ W["wv"].T
        T = h.shape[0]
        kk = k.reshape(T, cfg.n_kv, 1, cfg.head_dim).expand(T, cfg.n_kv, grp, cfg.head_dim).reshape(T, -1)
        vv = v.reshape(T, cfg.n_kv, 1, cfg.head_dim).expand(T, cfg.n_kv, grp, cfg.head_dim).reshape(T, -1)
        a = q + kk * vv
        x2 = h + a @ W["wo"].T
        h2 = rms(x2, W["mlp_norm"])
        g, u = h2 @ W["wgate"].T, h2 @ W["wup"].T
        h = x2 + (torch.nn.functional.silu(g) * u) @ W["wdown"].T
    loss = (0.5 * (h - torch.tensor(t, dtype=torch.float64)) ** 2).mean()
    loss.backward()
    return loss.item(), [{k: v.grad.numpy() for k, v in W.items()} for W in TW]


def test_llama_layer_fp64_vs_torch_autograd():
    """fp64 mode (no storage rounding) of the manual backward == autograd."""
    cfg = synth.small_llama(layers=2, seq=64)
    Ws = _small_weights(cfg)
    x, t = ost.rank_batch(cfg, 0)
    loss, G, _ = om.llama_stack_fwd_bwd(x, t, Ws, cfg, om.ident)
    tl, TG = _torch_stack(x, t, Ws, cfg)
    assert abs(loss - tl) <= 1e-12 * abs(tl)
    for l in range(cfg.layers):
        for k in G[l]:
            ref = TG[l][k]
            assert np.max(np.abs(G[l][k] - ref)) <= 1e-10 * np.max(np.abs(ref)), (l, k)


def test_llama_layer_bf16_close_to_fp64():
    cfg = synth.small_llama(layers=1, seq=128)
    Ws = _small_weights(cfg)
    x, t = ost.rank_batch(cfg, 0)
    xb = nx.rne_bf16(x)
    l64, G64, o64 = om.llama_stack_fwd_bwd(xb, t, Ws, cfg, om.ident)
    l16, G16, o16 = om.llama_stack_fwd_bwd(xb, t, Ws, cfg, nx.rne_bf16)
    assert abs(l16 - l64) <= 2e-2 * abs(l64)
    for k in G64[0]:
        a, b = G16[0][k], G64[0][k]
        assert np.linalg.norm(a - b) <= 2e-2 * np.linalg.norm(b), k


def test_llama_sharded_equals_unsharded_bitexact():
    cfg = synth.small_llama(layers=1, seq=64)
    table = synth.llama_param_table(cfg)
    N = 2
    sh = ost.ShardedState(table, N, bf16=True)
    rp = ost.ReplicatedState(table, N, bf16=True)
    for _ in range(2):
        l1, _ = ost.sharded_step(sh, cfg, lr=1.5e-5)
        l2 = ost.replicated_step(rp, cfg, lr=1.5e-5)
        assert l1 == l2
    for i, p in enumerate(table):
        got = nx.all_gather([sh.master[r][i] for r in range(N)], p.numel)
        assert got.tobytes() == rp.master[i].tobytes()


# ---------------------------------------------------------------- gradient accumulation
def test_micro_seeds_distinct_and_micro0_unchanged():
    assert synth.seed_inputs(3) == synth.seed_inputs(3, 0) == 1003
    seeds = {synth.seed_inputs(r, m) for r in range(8) for m in range(16)} | \
            {synth.seed_targets(r, m) for r in range(8) for m in range(16)}
    assert len(seeds) == 2 * 8 * 16


@pytest.mark.parametrize("n", [2, 3])
def test_mlp_accumulated_equals_full_batch(n):
    """n micro-steps x N ranks x b samples == the gradient of the mean loss over
    all N n b samples (§4.3: the update uses the gradient of
    the whole mini-batch), up to summation order.  A dropped 1/n, a missing
    micro-step or a double-counted one fails this."""
    cfg = synth.MLP_CONFIG1
    table = synth.mlp_param_table(cfg)
    N = 2
    full = ost.init_full_params(table)
    params = [(full[2 * l].reshape(256, 256), full[2 * l + 1]) for l in range(4)]
    xs, ts = zip(*[ost.rank_batch(cfg, r, m) for m in range(n) for r in range(N)])
    _, g_full = om.mlp_fwd_bwd(np.concatenate(xs), np.concatenate(ts), params)
    sh = ost.ShardedState(table, N, bf16=False)
    _, gp = ost.sharded_step(sh, cfg, lr=1e-3, micro_steps=n)
    for i, p in enumerate(table):
        red = np.concatenate([
            nx.scale_mean(nx.accumulate(sh.acc[r][i], nx.reduce_scatter([gp[q][i] for q in range(N)], N, r)),
                          N, n) for r in range(N)])[:p.numel]
        ref = (g_full[i // 2][i % 2]).reshape(-1)
        assert np.max(np.abs(red - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_accumulation_of_identical_micro_batches_is_exact():
    """Special case: n = 2 identical micro-batches give exactly the n = 1
    update (x + x is exact in fp32 and 1/(2N) is a power of two)."""
    g = synth.values(77, 0, 0, 1000, synth.K_UNIT)
    one = nx.scale_mean(g, 2, 1)
    two = nx.scale_mean(nx.accumulate(nx.accumulate(None, g), g), 2, 2)
    assert one.tobytes() == two.tobytes()


@pytest.mark.parametrize("kind", ["mlp", "llama"])
def test_sharded_equals_replicated_with_accumulation(kind):
    """§5.6 invariant with n = 2 micro-steps: per-micro RS + fp32 accumulation
    of the shard == per-micro all-reduce + accumulation of the full gradient."""
    if kind == "mlp":
        cfg, table, lr, bf = synth.MLP_CONFIG1, synth.mlp_param_table(synth.MLP_CONFIG1), 1e-3, False
    else:
        cfg = synth.small_llama(layers=1, seq=64)
        table, lr, bf = synth.llama_param_table(cfg), 1.5e-5, True
    N = 2
    sh = ost.ShardedState(table, N, bf16=bf)
    rp = ost.ReplicatedState(table, N, bf16=bf)
    for _ in range(2):
        l1, _ = ost.sharded_step(sh, cfg, lr=lr, micro_steps=2)
        l2 = ost.replicated_step(rp, cfg, lr=lr, micro_steps=2)
        assert l1 == l2
    for i, p in enumerate(table):
        got = nx.all_gather([sh.master[r][i] for r in range(N)], p.numel)
        assert got.tobytes() == rp.master[i].tobytes()


# ---------------------------------------------------------------- Mixtral-shaped layer (config 4)
def test_moe_routing_is_balanced_top2():
    """Fixed balanced top-2: every token goes to two distinct
    experts and every expert receives exactly 2 T / E tokens, ascending."""
    T, E = 96, 8
    e0, e1 = om.moe_route(T, E)
    assert np.all(e0 != e1)
    seen = np.zeros(T, int)
    for e in range(E):
        rows = om.expert_tokens(T, E, e)
        assert len(rows) == 2 * T // E and np.all(np.diff(rows) > 0)
        assert np.all((e0[rows] == e) | (e1[rows] == e))
        seen[rows] += 1
    assert np.all(seen == 2)


def _moe_weights(cfg, seed=7):
    table = synth.moe_param_table(cfg)
    full = ost.init_full_params(table)
    P = len(table) // cfg.layers
    Ws = []
    for l in range(cfg.layers):
        W = {}
        for j, p in enumerate(table[l * P:(l + 1) * P]):
            w = full[l * P + j].reshape(p.shape)
            if p.k == 0.0:
                w = w + synth.values(seed, p.id, 0, p.numel, 0.2)
            if p.name == "router":          # spread the gates away from 1/2
                w = w * 20.0
            W[p.name] = nx.rne_bf16(w)
        Ws.append(W)
    return Ws


def _torch_moe_stack(x, t, Ws, cfg):
    x = torch.tensor(x, dtype=torch.float64)
    TW = [{k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in W.items()} for W in Ws]

    def rms(z, g):
        return z * torch.rsqrt((z * z).mean(1, keepdim=True) + om.RMS_EPS) * g

    grp = cfg.n_heads // cfg.n_kv
    E = cfg.n_experts
    h = x
    for W in TW:
        T = h.shape[0]
        h1 = rms(h, W["attn_norm"])
        q, k, v = h1 @ W["wq"].T, h1 @ W["wk"].T, h1 @ W["wv"].T
        kk = k.reshape(T, cfg.n_kv, 1, cfg.head_dim).expand(T, cfg.n_kv, grp, cfg.head_dim).reshape(T, -1)
        vv = v.reshape(T, cfg.n_kv, 1, cfg.head_dim).expand(T, cfg.n_kv, grp, cfg.head_dim).reshape(T, -1)
        x2 = h + (q + kk * vv) @ W["wo"].T
        h2 = rms(x2, W["mlp_norm"])
        logits = h2 @ W["router"].T
        tok = torch.arange(T)
        sel = torch.stack([tok % E, (tok + 1) % E], 1)            # [T, 2]
        gates = torch.softmax(torch.gather(logits, 1, sel), dim=1)
        out = torch.zeros_like(x2)
        for e in range(E):
            for kslot in range(2):
                m = sel[:, kslot] == e
                xe = h2[m]
                oe = (torch.nn.functional.silu(xe @ W["w1_%d" % e].T) * (xe @ W["w3_%d" % e].T)) @ W["w2_%d" % e].T
                out = out.index_add(0, tok[m], gates[m, kslot:kslot + 1] * oe)
        h = x2 + out
    loss = (0.5 * (h - torch.tensor(t, dtype=torch.float64)) ** 2).mean()
    loss.backward()
    return loss.item(), [{k: v.grad.numpy() for k, v in W.items()} for W in TW]


def test_moe_layer_fp64_vs_torch_autograd():
    """fp64 mode of the manual Mixtral-shaped backward (gates, router, experts,
    scatter of dX) == torch.autograd fp64; a dropped term or wrong sign fails."""
    cfg = synth.small_mixtral(layers=2, seq=64)
    Ws = _moe_weights(cfg)
    x, t = ost.rank_batch(cfg, 0)
    loss, G, _ = om.llama_stack_fwd_bwd(x, t, Ws, cfg, om.ident)
    tl, TG = _torch_moe_stack(x, t, Ws, cfg)
    assert abs(loss - tl) <= 1e-12 * abs(tl)
    for l in range(cfg.layers):
        for k in G[l]:
            ref = TG[l][k]
            assert np.max(np.abs(G[l][k] - ref)) <= 1e-10 * np.max(np.abs(ref)), (l, k)


def test_moe_bf16_close_to_fp64_and_sharded_equals_replicated():
    cfg = synth.small_mixtral(layers=1, seq=64)
    Ws = _moe_weights(cfg)
    x, t = ost.rank_batch(cfg, 0)
    xb = nx.rne_bf16(x)
    l64, G64, _ = om.llama_stack_fwd_bwd(xb, t, Ws, cfg, om.ident)
    l16, G16, _ = om.llama_stack_fwd_bwd(xb, t, Ws, cfg, nx.rne_bf16)
    assert abs(l16 - l64) <= 2e-2 * abs(l64)
    for k in G64[0]:
        assert np.linalg.norm(G16[0][k] - G64[0][k]) <= 3e-2 * np.linalg.norm(G64[0][k]), k
    table = synth.moe_param_table(cfg)
    sh = ost.ShardedState(table, 2, bf16=True)
    rp = ost.ReplicatedState(table, 2, bf16=True)
    l1, _ = ost.sharded_step(sh, cfg, lr=1.5e-5)
    l2 = ost.replicated_step(rp, cfg, lr=1.5e-5)
    assert l1 == l2
    for i, p in enumerate(table):
        assert nx.all_gather([sh.master[r][i] for r in range(2)], p.numel).tobytes() == rp.master[i].tobytes()
