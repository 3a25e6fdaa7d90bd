"""Helpers to build planner profiles for tests (no method arithmetic here:
S_0 construction is delegated to the oracle under test / the C-ABI)."""
import random

import synth

from oracle import sched as osd

MB = 1000 * 1000


def affine_tc(latency_us, bytes_per_us):
    """T_c(V) = latency + V / bandwidth, as a 2-point piecewise-linear table."""
    return [[0, latency_us], [bytes_per_us, latency_us + 1]]


def make_profile(compute, B, pmem, transient=None, dur=None, tc=None, frags=None):
    """compute: list of (name, kind, phase, micro, layer, params);
    pmem: dict s0-index -> bytes or a callable(op) -> bytes."""
    ops = [dict(name=n, kind=k, phase=ph, micro=mu, layer=l, params=list(ps))
           for n, k, ph, mu, l, ps in compute]
    s0 = osd.build_s0(ops)
    for o in s0:
        o["p_mem"] = pmem(o) if callable(pmem) else pmem[o["id"]]
        o["transient"] = (transient(o) if callable(transient) else transient.get(o["id"], 0)) if transient else 0
        o["dur_us"] = (dur(o) if callable(dur) else dur.get(o["id"], 0)) if dur else 0
    params = [dict(id=p, bytes=b, layer=0) for p, b in sorted(B.items())]
    return dict(ops=s0, params=params, frags=frags or [], tc=tc or affine_tc(100, 40000))


def layered(L, n_micro=1, params_per_layer=1, ops_per_layer=1, with_rs=True):
    """A layered fwd+bwd compute graph: layer l owns params l*P..l*P+P-1."""
    P = params_per_layer
    comp = []
    for mu in range(n_micro):
        for l in range(L):
            for j in range(ops_per_layer):
                ps = [l * P + q for q in range(P)] if j == 0 else []
                comp.append(("f%d_%d" % (l, j), "compute", "fwd", mu, l, ps))
        for l in reversed(range(L)):
            for j in range(ops_per_layer):
                ps = [l * P + q for q in range(P)] if j == ops_per_layer - 1 else []
                comp.append(("b%d_%d" % (l, j), "compute", "bwd", mu, l, ps))
            if with_rs and mu == n_micro - 1:
                comp.append(("rs%d" % l, "rs", "bwd", mu, l, []))
    return comp


def random_profile(rng: random.Random, L=None, P=None, n_micro=1, frags=False):
    L = L or rng.randint(1, 4)
    P = P or rng.randint(1, 3)
    ops_per_layer = rng.randint(1, 3)
    comp = layered(L, n_micro, P, ops_per_layer)
    B = {p: rng.choice([1, 2, 4, 8, 16]) * 256 * rng.randint(1, 4) for p in range(L * P)}
    # activation memory rises through forward, falls through backward
    s0 = osd.build_s0([dict(name=n, kind=k, phase=ph, micro=mu, layer=l, params=list(ps))
                       for n, k, ph, mu, l, ps in comp])
    live = osd.live_before_s0(s0, B)
    base = rng.randint(0, 20000)
    act, pm, tr = base, {}, {}
    for o in s0:
        pm[o["id"]] = act + live[o["id"]]
        tr[o["id"]] = rng.choice([0, 0, 256, 1024]) if o["kind"] == "compute" else 0
        if o["kind"] == "compute":
            act += rng.randint(0, 3000) if o["phase"] == "fwd" else -rng.randint(0, 3000)
            act = max(act, base)
    fr = []
    if frags:
        for l in range(L):
            for s in range(2):
                fr.append(dict(id=len(fr), layer=l, bytes=rng.randint(1, 8) * 1024))
    tc = [[1024, rng.randint(5, 50)], [1 << 16, rng.randint(60, 200)], [1 << 20, rng.randint(300, 3000)]]
    prof = make_profile(comp, B, pm, tr, dur=lambda o: 10 if o["kind"] == "compute" else 0,
                        tc=tc, frags=fr)
    return prof


def a256(b):
    return (b + 255) // 256 * 256


def analytic_profile(cfg, N, op_ms, checkpoint=True, micro_steps=1):
    """S_0 profile of a synthetic layer stack at any size without a GPU: the
    executor's P_mem bookkeeping (model.cu compute_pmem: shard + master, two
    grad slots, workspace, inputs, saved activations of the layers between
    their forward op and the end of their backward, live gathered bytes under
    S_0; m / v as per-(layer, state) fragments, reading D14) and per-op
    durations from `op_ms` (ms per op name, recompute ops as their forward op).
    Returns (profile, shard elements per rank, B per param, params per layer)."""
    T, h, f = cfg.tokens, cfg.hidden, cfg.ffn
    qd, kvd = cfg.q_dim, cfg.kv_dim
    qkvd = qd + 2 * kvd
    table = synth.param_table(cfg)
    S = {p.id: -(-p.numel // (8 * N)) * 8 for p in table}
    B = {p.id: N * S[p.id] * 2 for p in table}
    E = sum(S.values())
    layers = {}
    for p in table:
        layers.setdefault(p.layer, []).append(p.id)
    grad_slot = max(sum(a256(B[i]) for i in ids) for ids in layers.values())
    piece = {"attn_norm": T * h * 2 + T * 4, "qkv": T * qkvd * 2, "attn_mix": T * qd * 2, "o_proj": T * h * 2,
             "mlp_norm": T * h * 2 + T * 4, "gate_up": T * 2 * f * 2, "act": T * f * 2, "down": T * h * 2}
    layer_set = sum(a256(v) for v in piece.values())
    ws = 2 * T * h * 2 + T * f * 2 + T * 2 * f * 2 + 2 * T * h * 2 + T * qkvd * 2 + (T // 16) * h * 4
    static = E * 6 + 2 * grad_slot + ws + 2 * micro_steps * T * h * 2 + (layer_set - T * h * 2 if checkpoint else 0)
    static += E * 4 if micro_steps > 1 else 0                      # fp32 grad accumulator
    comp = synth.compute_ops(cfg, micro_steps=micro_steps, checkpoint=checkpoint)
    s0 = osd.build_s0(comp)
    live = osd.live_before_s0(s0, B)
    act = 0
    held = {}
    for o in s0:
        o["p_mem"] = static + live[o["id"]] + act
        o["transient"] = 0
        nm = o["name"][3:] if o["name"].startswith("re_") else o["name"]
        head, _, tail = nm.rpartition("_")
        nm = head if tail.isdigit() else nm                    # exp_gu_3 -> exp_gu (per-expert ops)
        oname = o["name"].rpartition("_")[0] if o["name"].rpartition("_")[2].isdigit() else o["name"]
        if o["kind"] == "rs":
            o["dur_us"] = 1          # replaced below by the RS model
        elif o["kind"] == "compute":
            o["dur_us"] = max(1, int(round(op_ms.get(nm if o["phase"] == "fwd" else oname, 0.0) * 1000)))
            if o["name"].startswith("re_"):
                o["dur_us"] = max(1, int(round(op_ms.get(nm, 0.0) * 1000)))
        else:
            o["dur_us"] = 0
        if o["kind"] == "compute":
            if checkpoint:
                if o["phase"] == "fwd" and o["name"] == "down":
                    act += T * h * 2
                elif o["phase"] == "bwd" and o["name"] == "attn_norm_bwd":
                    act -= T * h * 2
            elif o["phase"] == "fwd":
                add = piece.get(o["name"], 0)
                held[(o["micro"], o["layer"])] = held.get((o["micro"], o["layer"]), 0) + add
                act += add
            elif o["name"] == "attn_norm_bwd":          # the layer's saved activations are freed
                act -= held.pop((o["micro"], o["layer"]), 0)
    # optimizer-state fragments (layer, m | v): they define M_opt, which passes
    # P and S add to P_mem (reading D14)
    frags = []
    for l, ids in sorted(layers.items()):
        for _ in range(2):
            frags.append(dict(id=len(frags), layer=l, bytes=4 * sum(S[i] for i in ids)))
    return dict(ops=s0, params=[dict(id=i, bytes=b, layer=0) for i, b in sorted(B.items())], frags=frags,
                tc=[]), E, B, layers
