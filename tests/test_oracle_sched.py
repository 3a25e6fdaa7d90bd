"""Pins for oracle/sched.py and oracle/sim.py.

Sources of truth (none of them the oracle itself):
* the Fig. 6 narrative of PAPER.md (line 285) — the D1 trace;
* SPEC.md's worked examples (S:125, S:126, S:142-148, S:183, S:231 corrected,
  S:284);
* closed forms (the fuse boundary bβ(2−α)/(2(α−1)));
* brute force: enumeration of every valid gather placement on tiny regions,
  an independent live-set memory walk, and interval-overlap checks.
"""
import itertools
import json
import random
from fractions import Fraction

import pytest

import synth
from oracle import sched as osd
from oracle.sim import simulate
from tests.sched_util import MB, affine_tc, make_profile, layered, random_profile

P, PS, PSO = osd.PASS_SHARD | osd.PASS_PREFETCH, osd.PASSES_PS, osd.PASSES_PS | osd.PASS_OFFLOAD
SHARD = osd.PASS_SHARD


def seq(plan):
    """(kind, members) per op — a readable trace of a planned schedule."""
    out = []
    for o in plan["ops"]:
        if o["kind"] in ("ag", "rel"):
            out.append((o["kind"], tuple(o["members"])))
        elif o["kind"] in ("compute", "rs"):
            out.append((o["kind"], o["id"]))
        else:
            out.append((o["kind"], o["members"][0]))
    return out


# ---------------------------------------------------------------- T_c and Fuse
def test_tc_examples():
    assert osd.tc_eval(affine_tc(100, 40000), 4 * MB) == 200
    assert osd.tc_eval([[1 * MB, 125], [2 * MB, 150]], 1_500_000) == Fraction(275, 2)
    assert osd.tc_eval([[1 * MB, 125], [2 * MB, 150]], 10) == 125                 # flat below
    assert osd.tc_eval([[1 * MB, 125], [2 * MB, 150]], 4 * MB) == 200             # extrapolated


def test_should_fuse_examples_and_closed_form():
    tc, a = affine_tc(100, 40000), (3, 2)
    assert osd.should_fuse(tc, 1 * MB, 1 * MB, a)          # 250 > 225
    assert not osd.should_fuse(tc, 4 * MB, 4 * MB, a)      # 400 <= 450
    assert osd.should_fuse(tc, 0, 0, a)                    # two latencies
    # boundary: V* = b*beta*(2-alpha)/(2(alpha-1)) = 40000*100*0.5/1 = 2,000,000 B
    lo, hi = 0, 10 * MB
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if osd.should_fuse(tc, mid, mid, a):
            lo = mid
        else:
            hi = mid
    assert lo == 1_999_999 and hi == 2_000_000


def test_fuse_groups():
    tc, a = affine_tc(100, 40000), (3, 2)
    U = [dict(id=i, params=[i]) for i in range(4)]
    assert osd.fuse(U, {0: MB, 1: MB, 2: MB, 3: MB}, tc, a) == [[(0, 0), (1, 1), (2, 2)], [(3, 3)]]
    assert osd.fuse(U[:2], {0: 4 * MB, 1: 4 * MB}, tc, a) == [[(0, 0)], [(1, 1)]]
    assert osd.fuse([], {}, tc, a) == []


# ---------------------------------------------------------------- S_0 (§4.1)
def test_s0_counts_and_adjacency():
    s0 = osd.build_s0([dict(name=n, kind=k, phase=ph, micro=mu, layer=l, params=list(ps))
                       for n, k, ph, mu, l, ps in layered(4)])
    assert sum(o["kind"] == "ag" for o in s0) == 8
    assert sum(o["kind"] == "rel" for o in s0) == 8
    for i, o in enumerate(s0):
        if o["kind"] == "ag":
            assert o["params"][0] in s0[i + 1]["params"]       # immediately before first use
        if o["kind"] == "rel":
            assert o["params"][0] in s0[i - 1]["params"]       # immediately after last use
    # multi-consumer: c1(p), c2(), c3(p) -> ag before c1, rel after c3
    s0 = osd.build_s0([dict(name="c%d" % i, kind="compute", phase="fwd", micro=0, layer=0, params=ps)
                       for i, ps in enumerate([[0], [], [0]])])
    assert [o["kind"] for o in s0] == ["ag", "compute", "compute", "compute", "rel"]
    # Llama-3 8B stack: 9 tensors x 32 layers x 2 phases gathers, 32 RS
    s0 = osd.build_s0(synth.models.llama_compute_ops(synth.LLAMA3_8B))
    assert sum(o["kind"] == "ag" for o in s0) == 576
    assert sum(o["kind"] == "rs" for o in s0) == 32
    # layer checkpointing: same gathers, but the backward gather of every
    # param except the down projection now lands before its recompute op
    s0c = osd.build_s0(synth.models.llama_compute_ops(synth.LLAMA3_8B, checkpoint=True))
    assert sum(o["kind"] == "ag" for o in s0c) == 576
    for i, o in enumerate(s0c):
        if o["kind"] == "ag" and o["phase"] == "bwd":
            nxt = next(x for x in s0c[i + 1:] if x["kind"] == "compute")
            assert nxt["name"].startswith("re_") or nxt["name"] == "down_bwd"
    # gradient accumulation: one RS per layer per micro-step
    s0g = osd.build_s0(synth.models.llama_compute_ops(synth.small_llama(layers=3), micro_steps=4))
    assert sum(o["kind"] == "rs" for o in s0g) == 12
    assert sum(o["kind"] == "ag" for o in s0g) == 9 * 3 * 2 * 4


# ---------------------------------------------------------------- Algorithm 1
def _fig6_profile(M_pf=10 ** 9):
    comp = [("c%d" % i, "compute", "fwd", 0, 0, [i]) for i in (1, 2, 3)] + [("end", "compute", "fwd", 0, 0, [])]
    pm = [10, 40, 45, 15, 50, 55, 25, 60, 65, 35]  # ag1 c1 rel1 ag2 c2 rel2 ag3 c3 rel3 end
    return make_profile(comp, {1: 30, 2: 30, 3: 30}, dict(enumerate(pm)))


def test_alg1_fig6_narrative_D1():
    """Fig. 6 (line 285): the first two gathers are prefetched at the beginning;
    the third is delayed until after the buffer of the first has been released."""
    plan = osd.plan(_fig6_profile(), 100, 10 ** 9, passes=P)
    assert seq(plan) == [("ag", (1,)), ("ag", (2,)), ("compute", 1), ("rel", (1,)), ("ag", (3,)),
                         ("compute", 4), ("rel", (2,)), ("compute", 7), ("rel", (3,)), ("compute", 9)]


def test_alg1_final_group_after_o1_D2():
    comp = [("ca", "compute", "fwd", 0, 0, []), ("cb", "compute", "fwd", 0, 0, []),
            ("cc", "compute", "fwd", 0, 0, [0]), ("end", "compute", "fwd", 0, 0, [])]
    pm = [85, 50, 50, 70, 90, 40]       # ca cb ag cc rel end
    plan = osd.plan(make_profile(comp, {0: 20}, dict(enumerate(pm))), 100, 10 ** 9, passes=P)
    assert [k for k, _ in seq(plan)][:3] == ["compute", "ag", "compute"]   # [ca, ag, cb, ...]


def test_alg1_faithful_vs_strict_D4():
    comp = [("c0", "compute", "fwd", 0, 0, []), ("ca", "compute", "fwd", 0, 0, []),
            ("cb", "compute", "fwd", 0, 0, []), ("cc", "compute", "fwd", 0, 0, [0]),
            ("end", "compute", "fwd", 0, 0, [])]
    pm = [40, 85, 50, 50, 70, 90, 40]   # c0 ca cb ag cc rel end
    prof = make_profile(comp, {0: 20}, dict(enumerate(pm)))
    faithful = osd.plan(prof, 100, 10 ** 9, passes=P, strict=False)
    strict = osd.plan(prof, 100, 10 ** 9, passes=P, strict=True)
    assert seq(faithful)[:4] == [("compute", 0), ("ag", (0,)), ("compute", 1), ("compute", 2)]
    assert seq(strict)[:4] == [("compute", 0), ("compute", 1), ("ag", (0,)), ("compute", 2)]
    assert faithful["peak_no_opt"] == 105 and strict["peak_no_opt"] == 85


def test_alg1_spec_example_corrected_D21():
    """S:231 with its arithmetic slip fixed: agC fails (60+50 >= 100) and stays;
    agB and agA join; latency-dominated T_c fuses them."""
    mk = lambda i, k, p=None: dict(id=i, kind=k, params=[p] if p is not None else [])
    reg = [mk(0, "compute"), mk(1, "ag", "A"), mk(2, "compute"), mk(3, "ag", "B"),
           mk(4, "compute"), mk(5, "ag", "C")]
    Pm = {0: 0, 1: 0, 2: 30, 3: 30, 4: 60, 5: 60}
    tr = {i: 0 for i in Pm}
    B = {"A": 30, "B": 30, "C": 50}
    tc = [[0, 1000], [10 ** 9, 1001]]           # latency dominated
    S = osd.alg1_region(reg, Pm, tr, B, 100, 1000, tc, (3, 2), strict=False)
    kinds = [(e["kind"], tuple(p for p, _ in e["members"]) if e["kind"] == "ag" else e["ref"]) for e in S]
    assert kinds == [("compute", 0), ("ag", ("A", "B")), ("compute", 2), ("compute", 4), ("ag", ("C",))]


def test_prefetch_group_bound():
    """Every group Algorithm 1 forms stays below M_prefetch."""
    comp = [("c%d" % i, "compute", "fwd", 0, 0, [i]) for i in range(6)] + [("end", "compute", "fwd", 0, 0, [])]
    B = {i: 300 for i in range(6)}
    prof = make_profile(comp, B, lambda o: 0)
    plan = osd.plan(prof, 10 ** 6, 1000, passes=P)
    for o in plan["ops"]:
        if o["kind"] == "ag":
            assert sum(B[p] for p in o["members"]) < 1000


# ---------------------------------------------------------------- simulator pin
def test_simulator_fig5_240_to_165():
    """16 layers, compute 10 ms, gather 5 ms: serial S_0 = 240 ms; prefetched
    with ample memory = 5 + 16*10 = 165 ms (Fig. 5)."""
    L, Bb = 16, 1 << 20
    comp = [("c%d" % l, "compute", "fwd", 0, l, [l]) for l in range(L)] + [("end", "compute", "fwd", 0, L, [])]
    prof = make_profile(comp, {l: Bb for l in range(L)}, lambda o: 0,
                        dur=lambda o: 10000 if o["kind"] == "compute" and o["params"] else 0,
                        tc=[[0, 0], [Bb, 5000]])
    s0 = osd.plan(prof, 10 ** 12, 10 ** 12, passes=SHARD)
    pf = osd.plan(prof, 10 ** 12, 10 ** 12, passes=P)
    assert simulate(s0["ops"], prof) == 240000
    assert simulate(pf["ops"], prof) == 165000


# ---------------------------------------------------------------- unsharding §4.3
def test_unshard_spec_example():
    """{1, 2, 8} MB with 4 MB above the peak -> {1 MB, 2 MB}."""
    sizes = {0: 8 * MB, 1: 1 * MB, 2: 2 * MB}
    comp = layered(3)
    prof = make_profile(comp, sizes, lambda o: 0)
    s0 = osd.build_s0([dict(name=n, kind=k, phase=ph, micro=mu, layer=l, params=list(ps))
                       for n, k, ph, mu, l, ps in comp])
    live = osd.live_before_s0(s0, sizes)
    for o in prof["ops"]:
        o["p_mem"] = live[o["id"]]
    plan = osd.plan(prof, 8 * MB + 4 * MB, 10 ** 12, passes=SHARD | osd.PASS_UNSHARD)
    assert plan["unshard"] == [1, 2]


def test_unshard_ga_count():
    """n=4 micro-steps, L=8, everything unsharded: 2*L*n = 64 gathers -> L = 8."""
    comp = layered(8, n_micro=4)
    prof = make_profile(comp, {p: 1024 for p in range(8)}, lambda o: 0)
    base = osd.plan(prof, 10 ** 12, passes=SHARD)
    assert sum(o["kind"] == "ag" for o in base["ops"]) == 64
    plan = osd.plan(prof, 10 ** 12, passes=SHARD | osd.PASS_UNSHARD)
    assert len(plan["unshard"]) == 8
    assert sum(o["kind"] == "ag" for o in plan["ops"]) == 8
    assert sum(o["bytes"] for o in plan["ops"] if o["kind"] == "ag") * 8 == \
        sum(o["bytes"] for o in base["ops"] if o["kind"] == "ag")


def test_unshard_affine_prefix_property():
    """Affine T_c, distinct sizes: the selection is a size-ascending prefix."""
    rng = random.Random(11)
    for _ in range(100):
        n = rng.randint(1, 6)
        sizes = rng.sample(range(1, 64), n)
        Bm = {p: s * 4096 for p, s in enumerate(sizes)}
        comp = layered(n)
        prof = make_profile(comp, Bm, lambda o: 0)
        budget = rng.randint(0, sum(Bm.values()))
        peak = max(Bm.values())
        sel = osd.plan(prof, peak + budget, passes=SHARD | osd.PASS_UNSHARD)["unshard"]
        asc = sorted(Bm, key=lambda p: Bm[p])
        assert sel == asc[:len(sel)]
        if len(sel) < n:
            assert sum(Bm[p] for p in sel) + Bm[asc[len(sel)]] > budget


# ---------------------------------------------------------------- Algorithm 2 §4.4
def _offload_profile(fwd_pm, bwd_pm, nfrag, fbytes):
    comp = [("o%d" % i, "compute", "fwd", 0, 0, []) for i in range(len(fwd_pm))]
    comp += [("b%d" % i, "compute", "bwd", 0, 0, []) for i in range(len(bwd_pm))]
    comp += [("rs0", "rs", "bwd", 0, 0, [])]
    pm = list(fwd_pm) + list(bwd_pm) + [bwd_pm[-1] if bwd_pm else 0]
    frags = [dict(id=i, layer=0, bytes=fbytes) for i in range(nfrag)]
    return make_profile(comp, {}, dict(enumerate(pm)), frags=frags)


def test_alg2_noop_when_fits():
    plan = osd.plan(_offload_profile([10, 20], [20, 10], 4, 10), 100, passes=PSO)
    assert plan["offload"] == [] and not any(o["kind"].startswith(("offload", "reload")) for o in plan["ops"])


def test_alg2_minimal_count():
    plan = osd.plan(_offload_profile([30, 60], [40], 6, 10), 100, passes=PSO)
    assert plan["offload"] == [0, 1]


def test_alg2_trace_and_reload():
    """P_mem {20, 50, 80}, M=100, M_opt=40 (4 x 10) -> two offloads, both
    synced before o3; the reloads start where the declining backward fits."""
    plan = osd.plan(_offload_profile([20, 50, 80], [60, 30], 4, 10), 100, passes=PSO)
    assert seq(plan) == [("offload", 0), ("offload", 1), ("compute", 0), ("compute", 1),
                         ("offload_sync", 0), ("offload_sync", 1), ("compute", 2),
                         ("reload", 1), ("reload", 0), ("compute", 3), ("compute", 4),
                         ("reload_sync", 1), ("reload_sync", 0), ("rs", 5)]
    assert plan["warnings"] == []


def test_reload_declining_profile():
    """decreasing backward memory -> each reload starts at the first op
    from which it fits to the end: 3 frags offloaded (90 + 40 - 30 = 100),
    resident 10; f2 fits from b1 (80+10+10), f1 from b2 (70+10+20), f0 from b3."""
    plan = osd.plan(_offload_profile([20, 50, 90], [90, 80, 70, 60, 10], 4, 10), 100, passes=PSO)
    assert plan["offload"] == [0, 1, 2]
    s = seq(plan)
    assert s[s.index(("reload", 2)) + 1] == ("compute", 4)
    assert s[s.index(("reload", 1)) + 1] == ("compute", 5)
    assert s[s.index(("reload", 0)) + 1] == ("compute", 6)
    # all equal backward memory -> the reloads cluster at one position
    plan = osd.plan(_offload_profile([20, 50, 90], [90, 40, 40, 40, 10], 4, 10), 100, passes=PSO)
    s = seq(plan)
    i = s.index(("reload", 2))
    assert s[i:i + 4] == [("reload", 2), ("reload", 1), ("reload", 0), ("compute", 4)]


def test_reload_flat_profile_sync_fallback():
    """flat P_mem = M through backward -> synchronous reload + warning."""
    plan = osd.plan(_offload_profile([20, 90], [90, 90], 2, 10), 100, passes=PSO)
    assert plan["warnings"] and all(w.startswith("reload_sync_fallback") for w in plan["warnings"])
    s = seq(plan)
    rs = s.index(("rs", 4))
    assert s[rs - 1][0] == "reload_sync" and ("reload", 0) in s[rs - 4:rs]


def test_reload_host_states_frees_after_update():
    """Reading D28 (host-resident fragments), hand trace.  Layers 1 then 0 in the
    backward; P_mem: a0 20, a1 80 | c1 80, rs1 60, c0 60, d0 40, rs0 40; frags
    f0 (layer 0), f1 (layer 1), 20 B each; M = 90 -> both offloaded (80 + 40 -
    40 <= 90), resident 0.  f1 (deadline rs1): c1 gives 80 + 20 > 90, rs1 gives
    60 + 20 -> reload before rs1.  f0 (deadline rs0): the paper's rule keeps f1
    counted (R = 20) after rs1, so f0 fits only from d0 (40 + 20 + 20 <= 90);
    host-resident f1 is written back after rs1, so f0 fits from c0 (60 + 20),
    not from rs1 (60 + 20 + 20 > 90)."""
    comp = [("a0", "compute", "fwd", 0, 0, []), ("a1", "compute", "fwd", 0, 1, []),
            ("c1", "compute", "bwd", 0, 1, []), ("rs1", "rs", "bwd", 0, 1, []),
            ("c0", "compute", "bwd", 0, 0, []), ("d0", "compute", "bwd", 0, 0, []), ("rs0", "rs", "bwd", 0, 0, [])]
    pm = dict(enumerate([20, 80, 80, 60, 60, 40, 40]))
    frags = [dict(id=0, layer=0, bytes=20), dict(id=1, layer=1, bytes=20)]
    prof = make_profile(comp, {}, pm, frags=frags)
    paper = seq(osd.plan(prof, 90, passes=PSO))
    host = seq(osd.plan(prof, 90, passes=PSO | osd.PASS_HOST_STATES))
    def before(s, f):       # the compute-like op a reload is issued in front of
        return next(e for e in s[s.index(("reload", f)):] if e[0] in ("compute", "rs"))
    for s in (paper, host):
        assert before(s, 1) == ("rs", 3)
    assert before(paper, 0) == ("compute", 5)
    assert before(host, 0) == ("compute", 4)
    assert osd.plan(prof, 90, passes=PSO | osd.PASS_HOST_STATES)["warnings"] == []


def test_alg2_infeasible():
    with pytest.raises(osd.Infeasible):
        osd.plan(_offload_profile([20, 120], [30], 2, 10), 100, passes=PSO)
    with pytest.raises(osd.Infeasible):
        osd.plan(_offload_profile([20, 95], [30], 2, 10), 100, passes=PS)


# ---------------------------------------------------------------- properties
def _check_plan(prof, plan, M, strict):
    B = {p["id"]: p["bytes"] for p in prof["params"]}
    s0 = prof["ops"]
    ops = plan["ops"]
    # structural: every consumer of p sees p gathered; never-later
    live, pos_of_ag = {}, {}
    for j, o in enumerate(ops):
        if o["kind"] == "ag":
            for p in o["members"]:
                assert p not in live
                live[p] = (o["arena_off"], osd.align256(B[p]))
        elif o["kind"] == "rel":
            assert o["members"][0] in live
            del live[o["members"][0]]
        elif o["kind"] in ("compute", "rs"):
            for p in s0[o["id"]]["params"]:
                assert p in live
    assert not live
    # arena: live intervals never overlap, all below capacity (independent walk)
    cur = {}
    for o in ops:
        if o["kind"] == "ag":
            off = o["arena_off"]
            for p in o["members"]:
                iv = (off, off + osd.align256(B[p]))
                for a, b in cur.values():
                    assert iv[1] <= a or iv[0] >= b
                assert iv[1] <= plan["capacity"]
                cur[p] = iv
                off += osd.align256(B[p])
        elif o["kind"] == "rel":
            cur.pop(o["members"][0])
    # ready flags: each gather's region was last freed by its waits_on release
    freed = []
    gid = {o["id"]: j for j, o in enumerate(ops) if o["kind"] == "ag"}
    relpos = {o["id"]: j for j, o in enumerate(ops) if o["kind"] == "rel"}
    for j, o in enumerate(ops):
        if o["kind"] == "rel":
            freed.append((j, o["arena_off"], o["arena_off"] + o["bytes"]))
        if o["kind"] == "ag":
            lo, hi = o["arena_off"], o["arena_off"] + o["bytes"]
            ov = [r for r, a, b in freed if a < hi and lo < b]
            if ov:
                assert o["waits_on"] == [ops[max(ov)]["id"]]
                assert o["id"] in ops[max(ov)]["posts_ready_for"]
            else:
                assert o["waits_on"] == []
    # independent memory walk (live-set from scratch)
    live0, lv = [], 0
    for o in s0:
        live0.append(lv)
        lv += B[o["params"][0]] if o["kind"] == "ag" else (-B[o["params"][0]] if o["kind"] == "rel" else 0)
    other = {o["id"]: o["p_mem"] - live0[o["id"]] for o in s0}
    peak, lv = 0, 0
    core = [o for o in ops if o["kind"] in ("compute", "rs", "ag", "rel")]
    for j, o in enumerate(core):
        nxt = next(x for x in core[j:] if x["kind"] in ("compute", "rs"))
        t = s0[o["id"]]["transient"] if o["kind"] in ("compute", "rs") else 0
        peak = max(peak, other[nxt["id"]] + lv + t)
        if o["kind"] == "ag":
            lv += sum(B[p] for p in o["members"])
        elif o["kind"] == "rel":
            lv -= B[o["members"][0]]
    assert peak == plan["peak_no_opt"]
    M_opt = sum(f["bytes"] for f in prof["frags"])
    base = max(o["p_mem"] + o["transient"] for o in s0)
    if strict and base + M_opt <= M:
        assert peak + M_opt <= M


def test_random_profiles_properties():
    rng = random.Random(1234)
    n_ok = 0
    for it in range(300):
        prof = random_profile(rng, n_micro=rng.choice([1, 1, 2]))
        base = max(o["p_mem"] + o["transient"] for o in prof["ops"])
        M = base + rng.randint(0, 40000)
        M_pf = rng.choice([2048, 8192, 1 << 30])
        for strict in (False, True):
            plan = osd.plan(prof, M, M_pf, passes=PS, strict=strict)
            _check_plan(prof, plan, M, strict)
            again = osd.plan(json.loads(json.dumps(prof)), M, M_pf, passes=PS, strict=strict)
            assert osd.canonical_json(plan) == osd.canonical_json(again)
            n_ok += 1
    assert n_ok == 600


def test_random_offload_minimality():
    rng = random.Random(99)
    hits = 0
    for it in range(200):
        prof = random_profile(rng, frags=True)
        base = max(o["p_mem"] + o["transient"] for o in prof["ops"])
        M_opt = sum(f["bytes"] for f in prof["frags"])
        M = base + rng.randint(0, M_opt)
        try:
            plan = osd.plan(prof, M, passes=PSO, strict=True)
        except osd.Infeasible:
            continue
        _check_plan(prof, plan, M + M_opt, strict=False)
        off = plan["offload"]
        fb = {f["id"]: f["bytes"] for f in prof["frags"]}
        if off:
            hits += 1
            # minimal prefix: dropping the last offloaded fragment violates the bound
            assert off == sorted(off) and off == list(range(len(off)))
            need = plan["peak_no_opt"]
            assert need + M_opt - sum(fb[i] for i in off) <= M
            assert need + M_opt - sum(fb[i] for i in off[:-1]) > M
            # every offloaded fragment: sync before reload, reload before its sync
            ks = [(o["kind"], o["members"][0]) for o in plan["ops"] if o["kind"] not in ("compute", "rs", "ag", "rel")]
            for f in off:
                assert ks.index(("offload", f)) < ks.index(("offload_sync", f)) < ks.index(("reload", f)) \
                    < ks.index(("reload_sync", f))
    assert hits > 20


def test_exhaustive_tiny_regions_strict_safe():
    """Enumerate every valid placement of the gathers of tiny forward regions
    (each gather anywhere before its consumer) and check, by brute force, that
    (1) Algorithm 1's strict output is one of them and within M whenever S_0
    is, (2) it never moves a gather later, (3) when some valid placement moves
    a gather earlier within M, strict output is not worse than S_0 in position
    sum (it does move gathers when a safe earlier slot exists)."""
    rng = random.Random(5)
    for it in range(60):
        n_c = rng.randint(2, 5)
        users = sorted(rng.sample(range(1, n_c), rng.randint(1, min(3, n_c - 1))))
        comp = [("c%d" % i, "compute", "fwd", 0, 0, [users.index(i)] if i in users else []) for i in range(n_c)]
        comp.append(("end", "compute", "fwd", 0, 0, []))
        B = {p: rng.randint(1, 5) * 10 for p in range(len(users))}
        s0 = osd.build_s0([dict(name=n, kind=k, phase=ph, micro=mu, layer=l, params=list(ps))
                           for n, k, ph, mu, l, ps in comp])
        live = osd.live_before_s0(s0, B)
        act = {}
        a = 0
        for o in s0:
            act[o["id"]] = a
            if o["kind"] == "compute":
                a += rng.randint(0, 30)
        prof = make_profile(comp, B, lambda o: act[o["id"]] + live[o["id"]])
        M = max(o["p_mem"] for o in prof["ops"]) + rng.randint(0, 60)
        plan = osd.plan(prof, M, 10 ** 9, passes=P, strict=True)
        comp_ids = [o["id"] for o in s0 if o["kind"] == "compute"]
        # brute force over slots: gather p issued before compute index k <= first use
        first_use = {p: comp_ids.index(next(o["id"] for o in s0 if o["kind"] == "compute" and p in o["params"]))
                     for p in B}
        best_ok = False
        for slots in itertools.product(*[range(first_use[p] + 1) for p in sorted(B)]):
            mem_ok = True
            for k, cid in enumerate(comp_ids):
                extra = sum(B[p] for p, s in zip(sorted(B), slots) if s <= k < first_use[p])
                # before compute k: prefetched gathers issued at slot <= k not yet at S_0 position
                if prof["ops"][cid]["p_mem"] + extra > M:
                    mem_ok = False
            if mem_ok and any(s < first_use[p] for p, s in zip(sorted(B), slots)):
                best_ok = True
        # planner's placement
        ops = plan["ops"]
        seen_c = 0
        slot = {}
        for o in ops:
            if o["kind"] == "compute":
                seen_c += 1
            if o["kind"] == "ag":
                for p in o["members"]:
                    slot[p] = seen_c
        for p in B:
            assert slot[p] <= first_use[p]                          # never later
        assert plan["peak_no_opt"] <= M                              # strict safety
        if not best_ok:
            assert all(slot[p] == first_use[p] for p in B)           # nothing safe to move


def test_reload_host_states_brute_force():
    """Reading D28 on random multi-layer profiles without gathers (so an op's
    memory is its P_mem + transient): for every reload placed without the
    synchronous fallback, (1) every backward op from the reload to its layer's
    RS fits, counting the resident state and every placed reload live there
    (a reload lives from its op to its RS), and (2) it is the earliest such
    op: one backward op earlier (when allowed) breaks the bound."""
    rng = random.Random(5)
    checked = 0
    for it in range(150):
        L = rng.randint(2, 4)
        comp = [("f%d" % l, "compute", "fwd", 0, l, []) for l in range(L)]
        for l in reversed(range(L)):
            comp += [("b%d_%d" % (l, j), "compute", "bwd", 0, l, []) for j in range(rng.randint(1, 3))]
            comp.append(("rs%d" % l, "rs", "bwd", 0, l, []))
        pm = {}
        for i, c in enumerate(comp):
            pm[i] = rng.randint(10, 60) if c[2] == "fwd" else rng.randint(5, 60)
        frags = [dict(id=2 * l + s, layer=l, bytes=rng.randint(5, 20)) for l in range(L) for s in range(2)]
        prof = make_profile(comp, {}, pm, frags=frags)
        M_opt = sum(f["bytes"] for f in frags)
        M = max(pm.values()) + rng.randint(0, M_opt)
        try:
            plan = osd.plan(prof, M, passes=PSO | osd.PASS_HOST_STATES)
        except osd.Infeasible:
            continue
        off = plan["offload"]
        if not off:
            continue
        fb = {f["id"]: f["bytes"] for f in frags}
        fl = {f["id"]: f["layer"] for f in frags}
        resident = M_opt - sum(fb[i] for i in off)
        ops = plan["ops"]
        # positions of compute-like ops in time order, and where each reload is issued
        pos, reload_at, rs_at = [], {}, {}
        pending = []
        for o in ops:
            if o["kind"] == "reload":
                pending.append(o["members"][0])
            elif o["kind"] in ("compute", "rs"):
                k = len(pos)
                pos.append(o["id"])
                for f in pending:
                    reload_at[f] = k
                pending = []
                if o["kind"] == "rs":
                    rs_at[prof["ops"][o["id"]]["layer"]] = k
        need = [prof["ops"][i]["p_mem"] + prof["ops"][i]["transient"] for i in pos]
        first_bwd = next(k for k, i in enumerate(pos) if prof["ops"][i]["phase"] == "bwd")
        fallback = {int(w.split("=")[1]) for w in plan["warnings"]}

        order = list(reversed(off))                     # reloads placed in this order
        for idx, f in enumerate(order):
            if f in fallback:
                continue
            lo, hi = reload_at[f], rs_at[fl[f]]
            placed = set(order[:idx])                   # reloads placed before f
            live_before = lambda k: sum(fb[g] for g in placed if reload_at[g] <= k <= rs_at[fl[g]])
            for k in range(lo, hi + 1):
                assert need[k] + resident + live_before(k) + fb[f] <= M, (it, f, k)
            prev = max([reload_at[g] for g in placed] + [first_bwd])
            if lo - 1 >= prev:
                assert any(need[k] + resident + live_before(k) + fb[f] > M for k in range(lo - 1, hi + 1)), (it, f)
            checked += 1
    assert checked > 100
