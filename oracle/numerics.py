"""Oracle numerics of the sharded-parameter life cycle.  TEST INFRASTRUCTURE ONLY.

PAPER.md §4.1 (line 236): "each parameter tensor is evenly partitioned across
all GPUs.  Before a layer is computed, each GPU gathers the required parameter
shards via an all-gather communication, reconstructing the full parameters
locally.  Once the layer computation is complete, the gathered parameters are
discarded."  PAPER.md §5.1 (line 440): bf16 mixed precision with FP32 copies of
parameters, gradients and Adam states.  Adam: PAPER.md line 127 / 370 (Kingma &
Ba); the update stays on the GPU (line 504).

Every floating-point operation below is an explicit IEEE fp32 operation on
numpy float32 scalars/arrays (no fused multiply-add anywhere), in the order
written, so the CUDA kernels can be held to it element by element.
"""
import numpy as np

F32 = np.float32


# ---------------------------------------------------------------------------
# bf16 (round-to-nearest-even) — the storage type of params/activations/grads
# ---------------------------------------------------------------------------
def bf16_bits(x):
    """fp32 -> bf16 bit pattern, round to nearest even (finite inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return b.astype(np.uint16)


def bf16_to_f32(bits):
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def rne_bf16(x):
    """Round to a bf16-representable fp32 value (fp64 inputs go through fp32)."""
    return bf16_to_f32(bf16_bits(np.asarray(x, dtype=np.float32)))


# ---------------------------------------------------------------------------
# Shard layout (§4.1: "evenly partitioned across all GPUs")
# ---------------------------------------------------------------------------
def shard_len(numel: int, world: int) -> int:
    """S_i = ceil(numel / (8N)) * 8 elements: even split, 16-byte aligned shards
    (8 elements), zero padding at the tail of the flat tensor."""
    return -(-numel // (8 * world)) * 8


def shard_of(full_flat, world: int, rank: int):
    """Rank r owns elements [r*S, (r+1)*S) of the zero-padded flat tensor."""
    full_flat = np.asarray(full_flat).reshape(-1)
    S = shard_len(full_flat.size, world)
    padded = np.zeros(world * S, dtype=full_flat.dtype)
    padded[:full_flat.size] = full_flat
    return padded[rank * S:(rank + 1) * S].copy()


def all_gather(shards, numel: int):
    """All-gather = concatenation of the N shards in rank order, padding dropped
    ("reconstructing the full parameters locally", line 236).  Bitwise copy."""
    return np.concatenate([np.asarray(s) for s in shards])[:numel]


def all_gather_padded(shards):
    """The unsharded buffer as the GPU arena holds it: N*S elements incl. padding."""
    return np.concatenate([np.asarray(s) for s in shards])


# ---------------------------------------------------------------------------
# Reduce-scatter (+1/N) — the gradient step of data parallelism (§2.1)
# ---------------------------------------------------------------------------
def reduce_scatter(grads_padded, world: int, rank: int):
    """Owner r receives sum_q grad_q[r*S:(r+1)*S], summed in fp32 in ascending
    rank order starting from +0.0f: (((0 + g_0) + g_1) + ... + g_{N-1})."""
    S = np.asarray(grads_padded[0]).size // world
    acc = np.zeros(S, dtype=F32)
    for q in range(world):
        acc = (acc + np.asarray(grads_padded[q][rank * S:(rank + 1) * S], dtype=F32)).astype(F32)
    return acc


def scale_mean(g, world: int, micro_steps: int = 1):
    """Data-parallel mean over N ranks and n accumulated micro-steps:
    g * fp32(1/(N n)), one rounding (exact for N n a power of two)."""
    return (g * F32(1.0 / (world * micro_steps))).astype(F32)


def accumulate(acc, rs):
    """Gradient accumulation of the partitioned fp32 gradient shard (ZeRO-3
    semantics): acc_0 = rs_0, acc_mu = acc_{mu-1} + rs_mu."""
    return np.asarray(rs, F32).copy() if acc is None else (acc + np.asarray(rs, F32)).astype(F32)


# ---------------------------------------------------------------------------
# Adam (Kingma & Ba) — torch single-tensor order, fp32 ops
# ---------------------------------------------------------------------------
def adam_scalars(step: int, lr: float, beta1: float, beta2: float):
    """Host-side scalars in fp64, each rounded once to fp32:
    s = lr / (1 - beta1^t),  c = sqrt(1 - beta2^t)."""
    bc1 = 1.0 - beta1 ** step
    bc2 = 1.0 - beta2 ** step
    return F32(lr / bc1), F32(np.sqrt(bc2))


def adam_update(p, m, v, g, step: int, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
    """One Adam step on fp32 arrays (weight decay 0).  Returns new (p, m, v).

        m <- m + (1-b1) * (g - m)
        v <- (b2 * v) + ((1-b2) * g) * g
        d <- sqrt(v) / c + eps
        p <- p + ((-s) * m) / d
    each arrow-step a sequence of correctly rounded fp32 ops, no FMA (the
    operand order of torch.optim.Adam's single-tensor CPU path, reading D18)."""
    p = np.asarray(p, F32); m = np.asarray(m, F32); v = np.asarray(v, F32); g = np.asarray(g, F32)
    w1 = F32(1.0 - beta1)
    w2 = F32(1.0 - beta2)
    b2 = F32(beta2)
    s, c = adam_scalars(step, lr, beta1, beta2)
    e = F32(eps)
    m_new = (m + (w1 * (g - m).astype(F32)).astype(F32)).astype(F32)
    v_new = ((b2 * v).astype(F32) + ((w2 * g).astype(F32) * g).astype(F32)).astype(F32)
    d = ((np.sqrt(v_new).astype(F32) / c).astype(F32) + e).astype(F32)
    p_new = (p + ((F32(-s) * m_new).astype(F32) / d).astype(F32)).astype(F32)
    return p_new, m_new, v_new


def rs_adam_shard(grads_bf16_padded, master, m, v, world, rank, step, lr, beta1=0.9,
                  beta2=0.999, eps=1e-8, acc=None, micro_steps=1):
    """What dc_reduce_scatter_step computes for one tensor on owner `rank` at
    the last micro-step: RS of bf16 grads summed in fp32, added to the
    accumulated shard of the earlier micro-steps (if any), x 1/(N n), Adam on
    the fp32 master/m/v shard, bf16 (RNE) param shard written back.
    Returns (master, m, v, shard_bf16)."""
    rs = reduce_scatter([np.asarray(x, F32) for x in grads_bf16_padded], world, rank)
    g = scale_mean(accumulate(acc, rs) if acc is not None else rs, world, micro_steps)
    p2, m2, v2 = adam_update(master, m, v, g, step, lr, beta1, beta2, eps)
    return p2, m2, v2, rne_bf16(p2)
