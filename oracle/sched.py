"""Oracle scheduler: DeepCompile's optimisation passes, step by step in the
paper's order and notation.  TEST INFRASTRUCTURE ONLY.

  build_s0      — §4.1 (line 251): AllGather just before a parameter's first
                  use, Release just after its last use, per (phase, micro-step)
                  region.
  alg1_region   — §4.2 Algorithm 1 (lines 312-337) with the readings D1-D6.
  fuse          — §4.2 (line 350): fuse two all-gathers iff
                  T_c(V1) + T_c(V2) > alpha * T_c(V1 + V2), folded left to right.
  select_unshard— §4.3 (lines 364-365): greedy by T_c(B_ag)/B_ag descending
                  while peak + sum B_ag <= M.
  alg2/reload   — §4.4 Algorithm 2 (lines 373-401) and the backward reload rule
                  (line 408).
  arena/flags   — the B200 build's symmetric-arena offsets (first fit) and the
                  ready-flag actions a push all-gather needs.

All arithmetic is exact: Python ints and fractions.Fraction; no floats.
The output is the canonical schedule JSON (keys sorted, no whitespace,
integers only) that dc_plan must reproduce byte for byte.
"""
import json
from fractions import Fraction

PASS_SHARD, PASS_PREFETCH, PASS_UNSHARD, PASS_OFFLOAD = 1, 2, 4, 8
PASS_HOST_STATES = 16     # reload rule for host-resident fragments (reading D28)
PASSES_PS = PASS_SHARD | PASS_PREFETCH | PASS_UNSHARD
GiB = 1 << 30


class ProfileError(ValueError):
    """Profile does not describe an S_0 (SPEC ProfileMismatch -> DC_EPROFILE)."""


class Infeasible(ValueError):
    """Memory limit cannot be met (SPEC Infeasible / InfeasibleBaseline ->
    DC_EINFEASIBLE)."""


def align256(b: int) -> int:
    return (b + 255) // 256 * 256


# ---------------------------------------------------------------------------
# §4.1 — the fully-sharded rewrite, S_0
# ---------------------------------------------------------------------------
def regions(ops):
    """Maximal runs of equal (phase, micro) — the scope of every pass (D6)."""
    out, cur, key = [], [], None
    for o in ops:
        k = (o["phase"], o["micro"])
        if cur and k != key:
            out.append(cur)
            cur = []
        cur.append(o)
        key = k
    if cur:
        out.append(cur)
    return out


def build_s0(compute_ops):
    """Insert AllGather(p) immediately before p's first consumer and Release(p)
    immediately after its last consumer, separately in every (phase, micro-step)
    region; several gathers/releases at one op in ascending param id.  Op ids are
    the positions in S_0."""
    out = []
    for reg in regions(compute_ops):
        first, last = {}, {}
        for i, o in enumerate(reg):
            for p in o["params"]:
                first.setdefault(p, i)
                last[p] = i
        for i, o in enumerate(reg):
            base = dict(phase=o["phase"], micro=o["micro"], layer=o["layer"])
            for p in sorted(p for p in first if first[p] == i):
                out.append(dict(base, kind="ag", params=[p], name="ag"))
            out.append(dict(o))
            for p in sorted(p for p in last if last[p] == i):
                out.append(dict(base, kind="rel", params=[p], name="rel"))
    for i, o in enumerate(out):
        o["id"] = i
    return out


# ---------------------------------------------------------------------------
# T_c(V): profiled communication time, piecewise linear (Table 1)
# ---------------------------------------------------------------------------
def tc_eval(tc, V):
    """Exact T_c(V) as a Fraction (µs).  Flat at the first point below it,
    linear between points, extrapolated with the last segment beyond."""
    b0, t0 = tc[0]
    if V <= b0 or len(tc) == 1:
        if V <= b0:
            return Fraction(t0)
        return Fraction(tc[-1][1])
    for j in range(len(tc) - 1):
        (ba, ta), (bb, tb) = tc[j], tc[j + 1]
        if V <= bb:
            return Fraction(ta) + Fraction((tb - ta) * (V - ba), bb - ba)
    (ba, ta), (bb, tb) = tc[-2], tc[-1]
    return Fraction(tb) + Fraction((tb - ta) * (V - bb), bb - ba)


def should_fuse(tc, V1, V2, alpha):
    """Line 350: T_c(V1) + T_c(V2) > alpha * T_c(V1 + V2), alpha = num/den."""
    an, ad = alpha
    return ad * (tc_eval(tc, V1) + tc_eval(tc, V2)) > an * tc_eval(tc, V1 + V2)


def fuse(U, B, tc, alpha):
    """Fuse(U) (line 348-350): fold left to right over U (time order); the
    running group absorbs the next gather iff should_fuse(V_run, V_next) (D7).
    Returns a list of groups, each a list of (param, s0_ag_id)."""
    groups, run, vrun = [], [], 0
    for o in U:
        p = o["params"][0]
        if run and should_fuse(tc, vrun, B[p], alpha):
            run.append((p, o["id"]))
            vrun += B[p]
        else:
            if run:
                groups.append(run)
            run, vrun = [(p, o["id"])], B[p]
    if run:
        groups.append(run)
    return groups


def _ag_entry(members):
    return dict(kind="ag", members=list(members))


def _from_s0(o):
    if o["kind"] == "ag":
        return _ag_entry([(o["params"][0], o["id"])])
    e = dict(kind=o["kind"], ref=o["id"])
    if o["kind"] == "rel":
        e["param"] = o["params"][0]
    return e


# ---------------------------------------------------------------------------
# §4.2 — Algorithm 1, proactive prefetching
# ---------------------------------------------------------------------------
def alg1_region(reg, Pm, tr, B, M, M_pf, tc, alpha, strict, log=None):
    """Algorithm 1 on one region, o_1..o_n = reg (S_0 order).

    for i = n .. 2:
      if o_i is allgather:
        m_U = sum B_ag(U + o_i);  m_{i-1} = P_mem(o_{i-1}) + m_U
        if m_{i-1} < M and m_U < M_prefetch:  U <- U + o_i
        else: S_f <- Fuse(U), U <- [], append S_f           (at o_i's slot, D3)
              then retry o_i as a new U; if that fails too, emit o_i in place (D1)
      else: append o_i           (strict mode first flushes U if U cannot stay
                                  live across o_i: P_mem + transient + sum B >= M, D4)
    Fuse(U) of the remainder goes right after o_1 (D2).
    Built in reverse, returned in time order."""
    n = len(reg)
    S_rev, U = [], []

    def emit_group():
        for g in reversed(fuse(U, B, tc, alpha)):
            S_rev.append(_ag_entry(g))

    def ok(i, mU):
        return Pm[reg[i - 1]["id"]] + mU < M and mU < M_pf

    for i in range(n - 1, 0, -1):
        o = reg[i]
        if o["kind"] == "ag":
            bo = B[o["params"][0]]
            mU = sum(B[u["params"][0]] for u in U) + bo
            if ok(i, mU):
                U.insert(0, o)
                if log is not None:
                    log.append(("join", o["id"], Pm[reg[i - 1]["id"]] + mU, mU))
            else:
                if U:
                    emit_group()
                U = []
                if ok(i, bo):
                    U = [o]
                    if log is not None:
                        log.append(("join", o["id"], Pm[reg[i - 1]["id"]] + bo, bo))
                else:
                    S_rev.append(_from_s0(o))
        else:
            if strict and U:
                if Pm[o["id"]] + tr[o["id"]] + sum(B[u["params"][0]] for u in U) >= M:
                    emit_group()
                    U = []
            S_rev.append(_from_s0(o))
    if U:
        emit_group()
    S_rev.append(_from_s0(reg[0]))
    return list(reversed(S_rev))


# ---------------------------------------------------------------------------
# Analytic re-profile (the inner loop of §3, done by replay — D11)
# ---------------------------------------------------------------------------
def live_before_s0(s0, B):
    """Bytes of gathered buffers live before each S_0 op."""
    live, out = 0, []
    for o in s0:
        out.append(live)
        if o["kind"] == "ag":
            live += B[o["params"][0]]
        elif o["kind"] == "rel":
            live -= B[o["params"][0]]
    return out


def entry_base(S, P_other):
    """Non-gather memory before each entry of S: compute-like entries carry
    their own P_other; a gather/release entry takes the P_other of the next
    compute-like entry (gathers and releases do not change other memory)."""
    out = [None] * len(S)
    nxt = None
    for j in range(len(S) - 1, -1, -1):
        e = S[j]
        if e["kind"] in ("compute", "rs"):
            nxt = P_other[e["ref"]]
        out[j] = nxt
    return out


def replay(S, P_other, tr, B):
    """mem_S(e) = P_other + live gathered bytes, before each entry; and the
    transient of each entry (compute-like only)."""
    base = entry_base(S, P_other)
    live, mem, trans = 0, [], []
    for j, e in enumerate(S):
        mem.append(base[j] + live)
        trans.append(tr[e["ref"]] if e["kind"] in ("compute", "rs") else 0)
        if e["kind"] == "ag":
            live += sum(B[p] for p, _ in e["members"])
        elif e["kind"] == "rel":
            live -= B[e["param"]]
    return mem, trans


def peak_of(S, P_other, tr, B):
    mem, trans = replay(S, P_other, tr, B)
    return max(m + t for m, t in zip(mem, trans)) if S else 0


# ---------------------------------------------------------------------------
# §4.3 — selective unsharding
# ---------------------------------------------------------------------------
def select_unshard(S, B, tc, peak, M):
    """Rank parameters with more than one gather by T_c(B)/B descending (ties:
    ascending id) and admit p iff peak + sum B_sel + B(p) <= M, skipping misfits
    and continuing (D9)."""
    count = {}
    for e in S:
        if e["kind"] == "ag":
            for p, _ in e["members"]:
                count[p] = count.get(p, 0) + 1
    cands = [p for p in sorted(count) if count[p] > 1]
    ratio = {p: tc_eval(tc, B[p]) / B[p] for p in cands}
    order = sorted(cands, key=lambda p: (-ratio[p], p))
    sel, tot = [], 0
    for p in order:
        if peak + tot + B[p] <= M:
            sel.append(p)
            tot += B[p]
    return sel


def apply_unshard(S, sel):
    """Keep p's first gather and last release; drop its other gathers (leaving
    the rest of a fused group intact) and other releases (D10)."""
    sel = set(sel)
    first_seen, last_rel = set(), {}
    for j, e in enumerate(S):
        if e["kind"] == "rel" and e["param"] in sel:
            last_rel[e["param"]] = j
    out = []
    for j, e in enumerate(S):
        if e["kind"] == "ag":
            mem = []
            for p, sid in e["members"]:
                if p in sel:
                    if p in first_seen:
                        continue
                    first_seen.add(p)
                mem.append((p, sid))
            if mem:
                out.append(_ag_entry(mem))
        elif e["kind"] == "rel" and e["param"] in sel and last_rel[e["param"]] != j:
            continue
        else:
            out.append(e)
    return out


# ---------------------------------------------------------------------------
# §4.4 — Algorithm 2 (forward offload) and the backward reload rule
# ---------------------------------------------------------------------------
def alg2_and_reload(S, P_other, tr, B, frags, M, s0, host_states=False):
    """Returns (S with offload entries, offloaded frag ids, warnings).

    Algorithm 2: M_peak = max mem(o); M_opt = sum B_os; offload fragments in
    ascending id while M_peak + M_opt - sum(offloaded) > M (OffloadStart at the
    front); walk the schedule and before op o, while mem(o) + M_opt - M^- > M,
    pop the FIFO front (D16), emit TransferSync+free, M^- += B_os.
    Reload (line 408): in reverse offload order, ReloadStart before the earliest
    backward op o (not before the previous reload, nor before the fragment's own
    free) such that every backward o' >= o satisfies
    mem(o') + (M_opt - M^-) + R + B_os <= M; TransferSync before the RS of the
    fragment's layer (D17).  No such o by that deadline -> synchronous reload
    there and a warning.

    host_states (reading D28): an offloaded fragment is on the device only from
    its reload to its layer's update (written back right after), so during the
    backward the resident state is M_opt - sum(offloaded) and a placed reload
    occupies only [its reload op, its RS op].  The earliest o (same lower
    bounds) such that every backward o' in [o, RS] satisfies
    mem(o') + resident + live(o') + B_os <= M, live(o') = bytes of the reloads
    already placed that span o'."""
    mem, trans = replay(S, P_other, tr, B)
    need = [m + t for m, t in zip(mem, trans)]
    M_opt = sum(f["bytes"] for f in frags)
    M_peak = max(need) if need else 0
    offl, tot = [], 0
    for f in sorted(frags, key=lambda f: f["id"]):
        if M_peak + M_opt - tot > M:
            offl.append(f)
            tot += f["bytes"]
    if M_peak + M_opt - tot > M:
        raise Infeasible("offloading every optimizer-state fragment does not fit M")
    if not offl:
        return S, [], []
    rs_pos = {}
    for j, e in enumerate(S):
        if e["kind"] == "rs":
            rs_pos[s0[e["ref"]]["layer"]] = j
    pre = [[] for _ in S]
    queue = list(offl)
    Mminus = 0
    freed_at = {}
    for j in range(len(S)):
        while need[j] + M_opt - Mminus > M:
            if not queue:
                raise Infeasible("memory exceeds M at op %d after all offloads" % j)
            f = queue.pop(0)
            if j > rs_pos.get(f["layer"], len(S)):
                raise Infeasible("fragment %d must be freed after its own update" % f["id"])
            pre[j].append(dict(kind="offload_sync", frag=f["id"], fbytes=f["bytes"]))
            Mminus += f["bytes"]
            freed_at[f["id"]] = j
    warnings = []
    # backward ops of the last micro-step
    phase_of = lambda e: s0[e["ref"]]["phase"] if "ref" in e else s0[e["members"][0][1]]["phase"]
    micro_of = lambda e: s0[e["ref"]]["micro"] if "ref" in e else s0[e["members"][0][1]]["micro"]
    last_micro = max(o["micro"] for o in s0)
    bwd = [j for j, e in enumerate(S) if phase_of(e) == "bwd" and micro_of(e) == last_micro]
    if not bwd:
        raise Infeasible("offloaded fragments need a backward region to reload in")
    suffix = [0] * (len(bwd) + 1)
    for k in range(len(bwd) - 1, -1, -1):
        suffix[k] = max(suffix[k + 1], need[bwd[k]])
    if host_states:
        resident = M_opt - tot
        live = [0] * len(bwd)
        prev = 0
        for f in reversed(offl):
            dead_j = rs_pos.get(f["layer"], bwd[-1])
            dead_k = bwd.index(dead_j) if dead_j in bwd else len(bwd) - 1
            lo = prev
            fj = freed_at.get(f["id"], -1)
            while lo < len(bwd) and bwd[lo] < fj:
                lo += 1
            k_sel = None
            for k in range(lo, dead_k + 1):
                if all(need[bwd[q]] + resident + live[q] + f["bytes"] <= M for q in range(k, dead_k + 1)):
                    k_sel = k
                    break
            if k_sel is None:
                warnings.append("reload_sync_fallback frag=%d" % f["id"])
                k_sel = dead_k
            for q in range(k_sel, dead_k + 1):
                live[q] += f["bytes"]
            pre[bwd[k_sel]].append(dict(kind="reload", frag=f["id"], fbytes=f["bytes"]))
            pre[dead_j].append(dict(kind="reload_sync", frag=f["id"], fbytes=f["bytes"]))
            prev = k_sel
        out = [dict(kind="offload", frag=f["id"], fbytes=f["bytes"]) for f in offl]
        for j, e in enumerate(S):
            out.extend(pre[j])
            out.append(e)
        return out, [f["id"] for f in offl], warnings
    resident = M_opt - Mminus
    R, prev = 0, 0
    for f in reversed(offl):
        dead_j = rs_pos.get(f["layer"], bwd[-1])
        dead_k = bwd.index(dead_j) if dead_j in bwd else len(bwd) - 1
        lo = prev
        fj = freed_at.get(f["id"], -1)
        while lo < len(bwd) and bwd[lo] < fj:
            lo += 1
        k_sel = None
        for k in range(lo, dead_k + 1):
            if suffix[k] + resident + R + f["bytes"] <= M:
                k_sel = k
                break
        if k_sel is None:
            warnings.append("reload_sync_fallback frag=%d" % f["id"])
            k_sel = dead_k
        pre[bwd[k_sel]].append(dict(kind="reload", frag=f["id"], fbytes=f["bytes"]))
        pre[dead_j].append(dict(kind="reload_sync", frag=f["id"], fbytes=f["bytes"]))
        R += f["bytes"]
        prev = k_sel
    out = [dict(kind="offload", frag=f["id"], fbytes=f["bytes"]) for f in offl]
    for j, e in enumerate(S):
        out.extend(pre[j])
        out.append(e)
    return out, [f["id"] for f in offl], warnings


# ---------------------------------------------------------------------------
# B200 build: symmetric-arena offsets (first fit) and ready-flag actions
# ---------------------------------------------------------------------------
def assign_arena(S, B):
    """Walk S in time order; a gather group takes the lowest offset where its
    256-byte-aligned members fit contiguously; each member's interval is freed at
    its Release.  Returns (capacity, {entry index: offset}, {entry index:
    member offset for releases}, {entry index: [interval]})."""
    alloc = {}          # param -> (off, size)
    cap = 0
    ag_off, rel_off, rel_iv = {}, {}, {}
    for j, e in enumerate(S):
        if e["kind"] == "ag":
            size = sum(align256(B[p]) for p, _ in e["members"])
            ivs = sorted(alloc.values())
            cand = [0] + [o + s for o, s in ivs]
            off = None
            for c in sorted(set(cand)):
                if all(c + size <= o or c >= o + s for o, s in ivs):
                    off = c
                    break
            ag_off[j] = off
            cur = off
            for p, _ in e["members"]:
                alloc[p] = (cur, align256(B[p]))
                cur += align256(B[p])
            cap = max(cap, off + size)
        elif e["kind"] == "rel":
            o, s = alloc.pop(e["param"])
            rel_off[j] = o
            rel_iv[j] = (o, s)
    return cap, ag_off, rel_off, rel_iv


def ready_flags(S, B, ag_off, rel_iv):
    """For each gather g: the latest earlier Release whose freed interval
    overlaps g's interval must have run on every receiving rank before any rank
    pushes into g's region (write-after-read across ranks).  None -> posted at
    step start."""
    waits, posts = {}, {j: [] for j in rel_iv}
    for j, e in enumerate(S):
        if e["kind"] != "ag":
            continue
        lo = ag_off[j]
        hi = lo + sum(align256(B[p]) for p, _ in e["members"])
        best = None
        for r in range(j):
            if r in rel_iv:
                o, s = rel_iv[r]
                if o < hi and lo < o + s:
                    best = r
        waits[j] = best
        if best is not None:
            posts[best].append(j)
    return waits, posts


# ---------------------------------------------------------------------------
# The whole planner
# ---------------------------------------------------------------------------
def validate_profile(prof):
    ops = prof["ops"]
    if not ops:
        raise ProfileError("empty profile")
    pids = {p["id"] for p in prof["params"]}
    for i, o in enumerate(ops):
        if o["id"] != i:
            raise ProfileError("op ids must be S_0 positions")
        if o["kind"] not in ("compute", "ag", "rel", "rs"):
            raise ProfileError("bad kind")
        if o["kind"] in ("ag", "rel") and len(o["params"]) != 1:
            raise ProfileError("gather/release must reference one param")
        for p in o["params"]:
            if p not in pids:
                raise ProfileError("unknown param")
        if o["p_mem"] < 0 or o["transient"] < 0 or o["dur_us"] < 0:
            raise ProfileError("negative profile value")
    if ops[-1]["kind"] not in ("compute", "rs"):
        raise ProfileError("last op must be compute-like")
    tc = prof["tc"]
    if not tc or any(tc[j][0] >= tc[j + 1][0] for j in range(len(tc) - 1)):
        raise ProfileError("tc table must be strictly increasing in bytes")
    # S_0 shape: rebuilding S_0 from the compute ops must give the same list
    comp = [dict(kind=o["kind"], phase=o["phase"], micro=o["micro"], layer=o["layer"],
                 params=list(o["params"]), name=o.get("name", "")) for o in ops
            if o["kind"] in ("compute", "rs")]
    s0 = build_s0(comp)
    sig = lambda o: (o["kind"], o["phase"], o["micro"], tuple(o["params"]))
    if [sig(o) for o in s0] != [sig(o) for o in ops]:
        raise ProfileError("profile is not an S_0 schedule")


def plan(prof, M, M_prefetch=2 * GiB, alpha=(3, 2), passes=PASSES_PS, strict=False):
    """dc_plan(profile, M): S_0 -> Algorithm 1 (+Fuse) -> unshard -> Algorithm 2
    + reload -> arena offsets -> flag actions.  Pass order fixed P -> S -> O
    (§4.5).  Returns the schedule as a dict (see canonical_json)."""
    validate_profile(prof)
    s0 = prof["ops"]
    B = {p["id"]: p["bytes"] for p in prof["params"]}
    tc = [tuple(x) for x in prof["tc"]]
    frags = prof.get("frags", [])
    M_opt = sum(f["bytes"] for f in frags)
    Pm = {o["id"]: o["p_mem"] for o in s0}
    tr = {o["id"]: o["transient"] for o in s0}
    live0 = live_before_s0(s0, B)
    P_other = {o["id"]: o["p_mem"] - live0[i] for i, o in enumerate(s0)}
    # Passes P and S see the optimizer state resident (profile after the outer
    # loop's warm-up, §3; D14).
    P_full = {k: v + M_opt for k, v in Pm.items()}
    base_peak = max(Pm[o["id"]] + tr[o["id"]] for o in s0)
    if not passes & PASS_OFFLOAD and base_peak + M_opt > M:
        raise Infeasible("S_0 peak %d + optimizer states %d exceed M %d" % (base_peak, M_opt, M))
    S = []
    for reg in regions(s0):
        if passes & PASS_PREFETCH:
            S += alg1_region(reg, P_full, tr, B, M, M_prefetch, tc, alpha, strict)
        else:
            S += [_from_s0(o) for o in reg]
    unshard = []
    if passes & PASS_UNSHARD:
        pk = peak_of(S, P_other, tr, B) + M_opt
        unshard = select_unshard(S, B, tc, pk, M)
        S = apply_unshard(S, unshard)
    offload, warnings = [], []
    if passes & PASS_OFFLOAD:
        S, offload, warnings = alg2_and_reload(S, P_other, tr, B, frags, M, s0,
                                               host_states=bool(passes & PASS_HOST_STATES))
    core = [e for e in S if e["kind"] in ("compute", "rs", "ag", "rel")]
    peak_no_opt = peak_of(core, P_other, tr, B)
    cap, ag_off, rel_off, rel_iv = assign_arena(S, B)
    waits, posts = ready_flags(S, B, ag_off, rel_iv)
    ops = []
    for j, e in enumerate(S):
        k = e["kind"]
        if k in ("compute", "rs"):
            ops.append(dict(kind=k, id=e["ref"], members=[], arena_off=-1, bytes=0,
                            waits_on=[], posts_ready_for=[]))
        elif k == "ag":
            ops.append(dict(kind=k, id=e["members"][0][1], members=[p for p, _ in e["members"]],
                            arena_off=ag_off[j],
                            bytes=sum(align256(B[p]) for p, _ in e["members"]),
                            waits_on=[] if waits[j] is None else [S[waits[j]]["ref"]],
                            posts_ready_for=[]))
        elif k == "rel":
            ops.append(dict(kind=k, id=e["ref"], members=[e["param"]], arena_off=rel_off[j],
                            bytes=align256(B[e["param"]]), waits_on=[],
                            posts_ready_for=[S[g]["members"][0][1] for g in posts[j]]))
        else:
            ops.append(dict(kind=k, id=-1, members=[e["frag"]], arena_off=-1,
                            bytes=e["fbytes"], waits_on=[], posts_ready_for=[]))
    return dict(capacity=cap, ops=ops, unshard=unshard, offload=offload,
                warnings=warnings, m_opt=M_opt, peak_no_opt=peak_no_opt)


def canonical_json(sched) -> str:
    """UTF-8, keys sorted, no whitespace, integers and ASCII strings only."""
    return json.dumps(sched, sort_keys=True, separators=(",", ":"))
