"""Oracle synthetic layer stacks and the N-rank simulated sharded step.
TEST INFRASTRUCTURE ONLY.

The paper's correctness claim (§5.6) is that the
sharded schedule trains the same model as ZeRO-3 — i.e. fully-sharded data
parallelism is an exact re-organisation of data parallelism (§2.1,
149; §4.1).  So the oracle of a step is the plain definition:

  sharded step  = per rank: all-gather -> forward -> backward -> grads;
                  reduce-scatter (fp32, rank order) -> x1/N -> Adam on the shard
  unsharded step = replicated data parallelism: full params on every rank,
                  all-reduce in the same rank order, Adam on the full tensor.

Both are elementwise-identical after the per-rank backward, so they must agree
bit for bit (tests/test_oracle_numerics.py).

Synthetic layer (shapes of PAPER.md line 440's Llama-3):
  h1 = RMSNorm(x)*g1;  q,k,v = h1 Wq^T, h1 Wk^T, h1 Wv^T
  a  = q + rep(k) * rep(v)        (token-local surrogate of attention, GQA rep)
  x2 = x + a Wo^T;  h2 = RMSNorm(x2)*g2
  y  = x2 + (SiLU(h2 Wg^T) * (h2 Wu^T)) Wd^T
Loss = mean 1/2 (y - t)^2 over the rank's elements.

`rnd` is the storage-rounding function applied at every GEMM / glue output:
numerics.rne_bf16 for the bf16 regime, identity for the fp64 pin mode (which is
checked against torch.autograd in fp64 so a dropped term or sign fails).
"""
import numpy as np


RMS_EPS = 1e-5


def ident(x):
    return np.asarray(x, dtype=np.float64)


def r64(rnd, x):
    return np.asarray(rnd(np.asarray(x, dtype=np.float64)), dtype=np.float64)


# ---------------------------------------------------------------------------
# RMSNorm and the surrogate attention mix
# ---------------------------------------------------------------------------
def rmsnorm_fwd(x, g, rnd):
    x = np.asarray(x, np.float64)
    rstd = 1.0 / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + RMS_EPS)
    n = x * rstd
    return r64(rnd, n * np.asarray(g, np.float64)[None, :]), rstd


def rmsnorm_bwd(dh, x, g, rstd):
    """d/dx and d/dg of h = x * rstd(x) * g (unrounded, fp64)."""
    x = np.asarray(x, np.float64); dh = np.asarray(dh, np.float64)
    g = np.asarray(g, np.float64)
    n = x * rstd
    dg = np.sum(dh * n, axis=0)
    dn = dh * g[None, :]
    dx = rstd * (dn - n * np.mean(dn * n, axis=1, keepdims=True))
    return dx, dg


def rep_kv(t, cfg):
    """[T, n_kv*hd] -> [T, n_heads*hd]: kv head j serves query heads
    j*(H/KV) .. (j+1)*(H/KV)-1 (grouped-query attention)."""
    T = t.shape[0]
    grp = cfg.n_heads // cfg.n_kv
    t3 = t.reshape(T, cfg.n_kv, 1, cfg.head_dim)
    return np.broadcast_to(t3, (T, cfg.n_kv, grp, cfg.head_dim)).reshape(T, cfg.q_dim)


def unrep_sum(t, cfg):
    """Adjoint of rep_kv: sum over the query heads of each kv group."""
    T = t.shape[0]
    grp = cfg.n_heads // cfg.n_kv
    return t.reshape(T, cfg.n_kv, grp, cfg.head_dim).sum(axis=2).reshape(T, cfg.kv_dim)


def silu(z):
    return z / (1.0 + np.exp(-z))


def dsilu(z):
    s = 1.0 / (1.0 + np.exp(-z))
    return s * (1.0 + z * (1.0 - s))


# ---------------------------------------------------------------------------
# Llama-shaped synthetic layer
# ---------------------------------------------------------------------------
def attn_fwd(x, W, cfg, rnd):
    """Attention half of the synthetic layer (shared by the Llama and Mixtral
    shapes): returns x2, h2 and the cache."""
    f = lambda k: np.asarray(W[k], np.float64)
    x = np.asarray(x, np.float64)
    h1, rstd1 = rmsnorm_fwd(x, f("attn_norm"), rnd)
    q = r64(rnd, h1 @ f("wq").T)
    k = r64(rnd, h1 @ f("wk").T)
    v = r64(rnd, h1 @ f("wv").T)
    a = r64(rnd, q + rep_kv(k, cfg) * rep_kv(v, cfg))
    x2 = r64(rnd, x + a @ f("wo").T)
    h2, rstd2 = rmsnorm_fwd(x2, f("mlp_norm"), rnd)
    return dict(x=x, h1=h1, rstd1=rstd1, q=q, k=k, v=v, a=a, x2=x2, h2=h2, rstd2=rstd2)


def attn_bwd(dy, dh2, c, W, cfg, rnd, G):
    """Backward of the attention half given dL/dy (through the residual) and
    dL/dh2 (through the MLP); fills G, returns dx."""
    f = lambda k: np.asarray(W[k], np.float64)
    dy = np.asarray(dy, np.float64)
    # h2 = RMSNorm(x2) * g2 ; x2 also feeds y directly
    dxn, dg2 = rmsnorm_bwd(dh2, c["x2"], f("mlp_norm"), c["rstd2"])
    G["mlp_norm"] = r64(rnd, dg2)
    dx2 = r64(rnd, dy + dxn)
    # x2 = x + a Wo^T
    da = r64(rnd, dx2 @ f("wo"))
    G["wo"] = r64(rnd, dx2.T @ c["a"])
    # a = q + rep(k) * rep(v)
    dq = da
    dk = r64(rnd, unrep_sum(da * rep_kv(c["v"], cfg), cfg))
    dv = r64(rnd, unrep_sum(da * rep_kv(c["k"], cfg), cfg))
    dh1 = r64(rnd, dq @ f("wq") + dk @ f("wk") + dv @ f("wv"))
    G["wq"] = r64(rnd, dq.T @ c["h1"])
    G["wk"] = r64(rnd, dk.T @ c["h1"])
    G["wv"] = r64(rnd, dv.T @ c["h1"])
    dxa, dg1 = rmsnorm_bwd(dh1, c["x"], f("attn_norm"), c["rstd1"])
    G["attn_norm"] = r64(rnd, dg1)
    return r64(rnd, dx2 + dxa)


def llama_layer_fwd(x, W, cfg, rnd):
    """W: dict name -> float array (bf16-valued for the bf16 regime)."""
    f = lambda k: np.asarray(W[k], np.float64)
    c = attn_fwd(x, W, cfg, rnd)
    h2 = c["h2"]
    gt = r64(rnd, h2 @ f("wgate").T)
    up = r64(rnd, h2 @ f("wup").T)
    act = r64(rnd, silu(gt) * up)
    y = r64(rnd, c["x2"] + act @ f("wdown").T)
    c.update(gt=gt, up=up, act=act)
    return y, c


def llama_layer_bwd(dy, c, W, cfg, rnd):
    """Returns dx and the parameter grads (rounded with rnd), manual backward."""
    f = lambda k: np.asarray(W[k], np.float64)
    dy = np.asarray(dy, np.float64)
    G = {}
    # y = x2 + act Wd^T
    dact = r64(rnd, dy @ f("wdown"))
    G["wdown"] = r64(rnd, dy.T @ c["act"])
    # act = silu(gt) * up
    dgt = r64(rnd, dact * c["up"] * dsilu(c["gt"]))
    dup = r64(rnd, dact * silu(c["gt"]))
    dh2 = r64(rnd, dgt @ f("wgate") + dup @ f("wup"))
    G["wgate"] = r64(rnd, dgt.T @ c["h2"])
    G["wup"] = r64(rnd, dup.T @ c["h2"])
    return attn_bwd(dy, dh2, c, W, cfg, rnd, G), G


# ---------------------------------------------------------------------------
# Mixtral-shaped layer: the MLP
# is replaced by E experts with fixed balanced top-2 routing.
#   logits = h2 Wr^T (fp32);  token t -> experts e0 = t mod E, e1 = (t+1) mod E
#   (g0, g1) = softmax(logits[t, e0], logits[t, e1])
#   expert e on its rows X_e = h2[tokens routed to e, ascending t]:
#     O_e = (SiLU(X_e W1_e^T) * (X_e W3_e^T)) W2_e^T
#   y[t] = x2[t] + g0[t] O_e0[t] + g1[t] O_e1[t]
# ---------------------------------------------------------------------------
def moe_route(T, E):
    """(e0, e1) per token of the fixed balanced top-2 routing."""
    e0 = np.arange(T) % E
    return e0, (e0 + 1) % E


def expert_tokens(T, E, e):
    """Tokens routed to expert e, ascending (every expert gets 2 T / E)."""
    e0, e1 = moe_route(T, E)
    return np.nonzero((e0 == e) | (e1 == e))[0]


def r32(x):
    """fp32 storage (router logits and gates are kept in fp32)."""
    return np.asarray(np.asarray(x, np.float64).astype(np.float32), np.float64)


def _gate_rnd(rnd):
    """fp32 rounding of router logits / gates in the storage-rounded regime;
    none in the fp64 pin mode (rnd = ident)."""
    return ident if rnd is ident else r32


def moe_layer_fwd(x, W, cfg, rnd):
    f = lambda k: np.asarray(W[k], np.float64)
    c = attn_fwd(x, W, cfg, rnd)
    h2, T, E, F = c["h2"], c["h2"].shape[0], cfg.n_experts, cfg.ffn
    r32 = _gate_rnd(rnd)
    logits = r32(h2 @ f("router").T)
    e0, e1 = moe_route(T, E)
    t = np.arange(T)
    l0, l1 = logits[t, e0], logits[t, e1]
    g0 = r32(1.0 / (1.0 + np.exp(l1 - l0)))
    g1 = r32(1.0 / (1.0 + np.exp(l0 - l1)))
    O = np.zeros((E, T, cfg.hidden))        # expert outputs scattered back to token rows
    exp_cache = []
    for e in range(E):
        rows = expert_tokens(T, E, e)
        X = h2[rows]
        gu = r64(rnd, X @ np.concatenate([f("w1_%d" % e), f("w3_%d" % e)]).T)
        a, b = gu[:, :F], gu[:, F:]
        H = r64(rnd, silu(a) * b)
        O[e, rows] = r64(rnd, H @ f("w2_%d" % e).T)
        exp_cache.append(dict(rows=rows, X=X, a=a, b=b, H=H))
    y = r64(rnd, c["x2"] + g0[:, None] * O[e0, t] + g1[:, None] * O[e1, t])
    c.update(logits=logits, g0=g0, g1=g1, O=O, exp=exp_cache)
    return y, c


def moe_layer_bwd(dy, c, W, cfg, rnd):
    f = lambda k: np.asarray(W[k], np.float64)
    dy = np.asarray(dy, np.float64)
    G = {}
    h2, T, E, F = c["h2"], dy.shape[0], cfg.n_experts, cfg.ffn
    r32 = _gate_rnd(rnd)
    e0, e1 = moe_route(T, E)
    t = np.arange(T)
    g0, g1, O = c["g0"], c["g1"], c["O"]
    # combine: dO_e[t] = g_k[t] dy[t] for the pair (t, e = e_k); dg_k = <dy, O_e_k>
    dO = np.zeros_like(O)
    dO[e0, t] = r64(rnd, g0[:, None] * dy)
    dO[e1, t] = r64(rnd, g1[:, None] * dy)
    dg0 = r32(np.sum(dy * O[e0, t], axis=1))
    dg1 = r32(np.sum(dy * O[e1, t], axis=1))
    dX = np.zeros((E, T, cfg.hidden))
    for e in range(E):
        ec = c["exp"][e]
        rows = ec["rows"]
        dOe = dO[e, rows]
        dH = r64(rnd, dOe @ f("w2_%d" % e))
        G["w2_%d" % e] = r64(rnd, dOe.T @ ec["H"])
        da = r64(rnd, dH * ec["b"] * dsilu(ec["a"]))
        db = r64(rnd, dH * silu(ec["a"]))
        dX[e, rows] = r64(rnd, da @ f("w1_%d" % e) + db @ f("w3_%d" % e))
        G["w1_%d" % e] = r64(rnd, da.T @ ec["X"])
        G["w3_%d" % e] = r64(rnd, db.T @ ec["X"])
    # gates: g0 = sigma(l0 - l1), g1 = 1 - g0  ->  dl0 = g0 g1 (dg0 - dg1), dl1 = -dl0
    dl0 = r32(g0 * g1 * (dg0 - dg1))
    dlog = np.zeros((T, E))
    dlog[t, e0] = dl0
    dlog[t, e1] = -dl0
    G["router"] = r64(rnd, dlog.T @ h2)
    dh2 = r64(rnd, dX[e0, t] + dX[e1, t] + dlog @ f("router"))
    return attn_bwd(dy, dh2, c, W, cfg, rnd, G), G


def mse_loss(y, t):
    """Loss = mean over the rank's elements of 1/2 (y - t)^2 and dL/dy."""
    y = np.asarray(y, np.float64); t = np.asarray(t, np.float64)
    d = y - t
    return float(np.mean(0.5 * d * d)), d / d.size


def llama_stack_fwd_bwd(x, t, Ws, cfg, rnd):
    """Ws: list over layers of weight dicts.  Returns (loss, grads per layer,
    layer outputs).  Mixtral-shaped layers when cfg.n_experts > 0."""
    layer_fwd, layer_bwd = (moe_layer_fwd, moe_layer_bwd) if cfg.n_experts else (llama_layer_fwd, llama_layer_bwd)
    h = r64(rnd, x)
    caches, outs = [], []
    for W in Ws:
        h, c = layer_fwd(h, W, cfg, rnd)
        caches.append(c)
        outs.append(h)
    loss, dy = mse_loss(h, t)
    d = r64(rnd, dy)
    grads = [None] * len(Ws)
    for l in reversed(range(len(Ws))):
        d, grads[l] = layer_bwd(d, caches[l], Ws[l], cfg, rnd)
    return loss, grads, outs


# ---------------------------------------------------------------------------
# MLP config 1 (fp32): 4 x Linear(256,256)+bias, ReLU between
# ---------------------------------------------------------------------------
def mlp_fwd_bwd(x, t, params):
    """params: list of (W[out,in], b[out]) fp32.  Returns (loss, grads[(dW, db)]).
    All math in fp32 numpy (the regime of BASELINE config 1)."""
    F = np.float32
    hs = [np.asarray(x, F)]
    zs = []
    for l, (W, b) in enumerate(params):
        z = (hs[-1] @ W.T + b).astype(F)
        zs.append(z)
        hs.append(np.maximum(z, F(0)) if l < len(params) - 1 else z)
    y = hs[-1]
    d = (y - np.asarray(t, F)).astype(F)
    loss = float(np.mean(F(0.5) * d * d, dtype=np.float64))
    dz = (d / F(d.size)).astype(F)
    grads = [None] * len(params)
    for l in reversed(range(len(params))):
        W, _ = params[l]
        if l < len(params) - 1:
            dz = np.where(zs[l] > 0, dz, F(0)).astype(F)
        grads[l] = ((dz.T @ hs[l]).astype(F), dz.sum(axis=0, dtype=F).astype(F))
        dz = (dz @ W).astype(F)
    return loss, grads
