"""N-rank simulated training steps (sharded and replicated).  TEST INFRASTRUCTURE ONLY.

A single process simulates N ranks ("Oracle").  The sharded step
follows the per-layer life cycle of PAPER.md §4.1 (line 236) and the update of
§4.4 / §5.4 (Adam kept on the GPU, line 504); the replicated step is plain data
parallelism (§2.1).
"""
import numpy as np

import synth
from . import numerics as nx
from . import model as om

F32 = np.float32


def init_full_params(table):
    """Full fp32 master tensors from the counter-based generator (synth.gen);
    norm gains (k == 0) are exactly 1.0."""
    out = []
    for p in table:
        if p.k == 0.0:
            out.append(np.ones(p.numel, dtype=F32))
        else:
            out.append(synth.values(synth.SEED_WEIGHTS, p.id, 0, p.numel, p.k))
    return out


def rank_batch(cfg, rank, micro=0):
    """Rank r's synthetic micro-batch `micro` (inputs std 1, targets std 1)."""
    n = cfg.tokens * cfg.hidden
    x = synth.values(synth.seed_inputs(rank, micro), 0, 0, n, synth.K_UNIT).reshape(cfg.tokens, cfg.hidden)
    t = synth.values(synth.seed_targets(rank, micro), 0, 0, n, synth.K_UNIT).reshape(cfg.tokens, cfg.hidden)
    return x, t


class ShardedState:
    """Per rank: fp32 master / m / v shards and the storage-dtype param shard."""

    def __init__(self, table, world, bf16):
        self.table, self.world, self.bf16 = table, world, bf16
        full = init_full_params(table)
        self.S = [nx.shard_len(p.numel, world) for p in table]
        self.master = [[nx.shard_of(full[i], world, r) for i in range(len(table))] for r in range(world)]
        self.m = [[np.zeros(self.S[i], F32) for i in range(len(table))] for r in range(world)]
        self.v = [[np.zeros(self.S[i], F32) for i in range(len(table))] for r in range(world)]
        self.shard = [[(nx.rne_bf16(x) if bf16 else x.copy()) for x in self.master[r]] for r in range(world)]
        self.t = 0

    def gathered(self, rank):
        """All-gather of every param as seen by `rank` (identical on all ranks)."""
        return [nx.all_gather([self.shard[q][i] for q in range(self.world)], p.numel)
                for i, p in enumerate(self.table)]


def _fwd_bwd(cfg, table, full, x, t, bf16):
    if cfg.kind == "mlp":
        params = [(full[2 * l].reshape(cfg.hidden, cfg.hidden), full[2 * l + 1]) for l in range(cfg.layers)]
        loss, grads = om.mlp_fwd_bwd(x, t, params)
        flat = []
        for dW, db in grads:
            flat += [dW.reshape(-1), db.reshape(-1)]
        return loss, flat, None
    # llama-shaped, bf16 regime
    rnd = nx.rne_bf16 if bf16 else om.ident
    names = [p.name for p in table[:len(table) // cfg.layers]]
    P = len(names)
    Ws = [{p.name: full[l * P + j].reshape(p.shape) for j, p in enumerate(table[l * P:(l + 1) * P])}
          for l in range(cfg.layers)]
    # bf16 regime: inputs and targets are stored in bf16 like every activation
    loss, G, outs = om.llama_stack_fwd_bwd(nx.rne_bf16(x) if bf16 else x, nx.rne_bf16(t) if bf16 else t,
                                           Ws, cfg, rnd)
    flat = []
    for l in range(cfg.layers):
        for nm in names:
            flat.append(np.asarray(G[l][nm], F32).reshape(-1))
    return loss, flat, outs


def sharded_step(state: ShardedState, cfg, lr, micro_steps=1):
    """One sharded optimizer step over all simulated ranks with n micro-steps
    (§4.3: n forward/backward passes, then one update).
    Every micro-step's bf16 grads are reduce-scattered (fp32, rank order) and
    accumulated into the partitioned fp32 gradient shard; the last micro-step
    applies x 1/(N n) and Adam.  Returns per-rank losses (of the last
    micro-step) and the last micro-step's padded grads (grad-slot contents)."""
    N = state.world
    state.t += 1
    acc = [[None] * len(state.table) for _ in range(N)]
    state.micro_losses = []     # [micro][rank]
    for mu in range(micro_steps):
        losses, grads_padded = [], []
        for r in range(N):
            full = state.gathered(r)
            x, t = rank_batch(cfg, r, mu)
            loss, flat, _ = _fwd_bwd(cfg, state.table, full, x, t, state.bf16)
            losses.append(loss)
            grads_padded.append([np.concatenate([g, np.zeros(N * state.S[i] - g.size, F32)])
                                 for i, g in enumerate(flat)])
        state.micro_losses.append(losses)
        if mu < micro_steps - 1:
            for r in range(N):
                for i in range(len(state.table)):
                    rs = nx.reduce_scatter([grads_padded[q][i] for q in range(N)], N, r)
                    acc[r][i] = nx.accumulate(acc[r][i], rs)
    state.acc = acc          # accumulated shards of micro-steps 0..n-2 (tests inspect it)
    for r in range(N):
        for i in range(len(state.table)):
            mst, m, v, sh = nx.rs_adam_shard([grads_padded[q][i] for q in range(N)],
                                             state.master[r][i], state.m[r][i], state.v[r][i],
                                             N, r, state.t, lr, acc=acc[r][i], micro_steps=micro_steps)
            state.master[r][i], state.m[r][i], state.v[r][i] = mst, m, v
            state.shard[r][i] = sh if state.bf16 else mst.copy()
    return losses, grads_padded


class ReplicatedState:
    """Plain data parallelism: every rank holds the full fp32 params and states."""

    def __init__(self, table, world, bf16):
        self.table, self.world, self.bf16 = table, world, bf16
        self.master = init_full_params(table)
        self.m = [np.zeros(p.numel, F32) for p in table]
        self.v = [np.zeros(p.numel, F32) for p in table]
        self.t = 0

    def params(self):
        return [nx.rne_bf16(x) if self.bf16 else x for x in self.master]


def replicated_step(state: ReplicatedState, cfg, lr, micro_steps=1):
    """Plain data parallelism: per micro-step an all-reduce (fp32, ascending
    rank from +0.0) accumulated over micro-steps, x 1/(N n), Adam on the full
    tensors."""
    N = state.world
    state.t += 1
    full = state.params()
    total = [None] * len(state.table)
    for mu in range(micro_steps):
        per_rank, losses = [], []
        for r in range(N):
            x, t = rank_batch(cfg, r, mu)
            loss, flat, _ = _fwd_bwd(cfg, state.table, full, x, t, state.bf16)
            losses.append(loss)
            per_rank.append(flat)
        for i in range(len(state.table)):
            ar = np.zeros(state.table[i].numel, F32)
            for q in range(N):
                ar = (ar + per_rank[q][i]).astype(F32)
            total[i] = nx.accumulate(total[i], ar)
    for i in range(len(state.table)):
        g = nx.scale_mean(total[i], N, micro_steps)
        state.master[i], state.m[i], state.v[i] = nx.adam_update(
            state.master[i], state.m[i], state.v[i], g, state.t, lr)
    return losses
