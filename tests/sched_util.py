"""Helpers to build planner profiles for tests (no method arithmetic here:
S_0 construction is delegated to the oracle under test / the C-ABI)."""
import random

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
