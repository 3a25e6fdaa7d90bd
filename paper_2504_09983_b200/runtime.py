"""Torch-side plumbing around the C ABI: allocate the shard store, the
symmetric grad slots / flag tables / gather arena, the activation buffer and the
streams, then drive profile -> plan -> step through libdc_b200.so.

Two ways to get N ranks:
  * one process per GPU (torchrun): peer pointers from torch symmetric memory
    (`torch.distributed._symmetric_memory.empty` + `rendezvous`);
  * DC_VIRTUAL_RANKS: N ranks on one GPU in one process, each with its own
    buffers; the "peer" pointers are the other virtual ranks' device buffers.
    Every rank's host calls run in their own thread (one ctx per thread).
Nothing here computes: all math runs in the library's kernels.
"""
import ctypes as C
import json
import os
import threading

import torch

from . import dc

GiB = 1 << 30


def table_arrays(table):
    return ([p.numel for p in table], [p.layer for p in table], [float(p.k) for p in table])


def max_s0_ops(table, micro_steps=1):
    # one gather and one release per param per phase, the compute ops (at most
    # 3 per param and 20 per layer, incl. recompute) + RS per layer, per
    # micro-step, rounded up generously
    return (8 * len(table) + 24 * (max(p.layer for p in table) + 1) + 16) * micro_steps


class RankState:
    """One rank's buffers, context, model and streams."""

    def __init__(self):
        self.ctx = None
        self.model = None
        self.tensors = {}
        self.peer_keep = {}     # per symmetric buffer: imported peer mappings (IPC storages / symm_mem handle)
        self.nvls = None        # what bind_multicast selected (N > 1, DC_NVLS)
        self.streams = None
        self.aux_streams = []    # virtual ranks: the model's dW / write-back streams (from the pool)
        self.sched = None
        self.micro_steps = 1

    def stream_handles(self):
        return [s.cuda_stream for s in self.streams]


def _alloc_symmetric_ipc(nbytes, group, device):
    """Peer-mapped buffer through CUDA IPC: every rank exports its allocation's
    IPC handle over the process group and opens the others' (works between
    processes on one device, and across NVLink-connected devices).  Returns
    (local tensor, peer pointers, keep): `keep` holds the imported peer
    storages and must outlive every use of their pointers."""
    import torch.distributed as dist
    t = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if dist.get_world_size(group) == 1:          # nothing to export
        return t, [t.data_ptr()], []
    h = t.untyped_storage()._share_cuda_()
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, h, group=group)
    me = dist.get_rank(group)
    ptrs, keep = [], []
    for q, hq in enumerate(handles):
        if q == me:
            ptrs.append(t.data_ptr())
        else:
            st = torch.UntypedStorage._new_shared_cuda(*hq)
            keep.append(st)
            ptrs.append(st.data_ptr())
    return t, ptrs, keep


def symm_backend():
    """Which peer-mapping path _alloc_symmetric uses: "symm_mem" (torch
    symmetric memory, the default for one process per GPU) or "ipc" (CUDA IPC,
    DC_SYMM=ipc — required when several processes share one GPU, which
    symmetric memory refuses).  If torch symmetric memory was tried without an
    explicit DC_SYMM and refused, "ipc (torch symmetric memory unavailable:
    <reason>)" — the fallback is reported, never silent."""
    v = os.environ.get("DC_SYMM", "symm_mem")
    if v not in ("symm_mem", "ipc"):
        raise ValueError("DC_SYMM must be symm_mem or ipc, got %r" % v)
    if v == "symm_mem" and SYMM_FALLBACK:
        return "ipc (torch symmetric memory unavailable: %s)" % SYMM_FALLBACK
    return v


SYMM_FALLBACK = None     # reason torch symmetric memory was not used (recorded, reported by bench.py)


def _alloc_symmetric(nbytes, group, device):
    """Symmetric buffer for the peer tables (grad slots, flags, gather arena).
    Returns (local tensor, [world] peer pointers, keep-alive handles).  With
    DC_SYMM set explicitly the chosen backend must work (raises otherwise).
    Without it, torch symmetric memory is tried and, if the runtime refuses it,
    CUDA IPC is used LOUDLY: a warning on stderr and the reason in
    SYMM_FALLBACK, which bench.py puts in its JSON line (collectives.transport)
    — never a silent switch of what the N > 1 numbers measure."""
    global SYMM_FALLBACK
    if symm_backend() == "ipc" or SYMM_FALLBACK:
        return _alloc_symmetric_ipc(nbytes, group, device)
    try:
        from torch.distributed import _symmetric_memory as symm_mem
        t = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
        h = symm_mem.rendezvous(t, group)
    except Exception as e:     # noqa: BLE001 - recorded and reported, see above
        if os.environ.get("DC_SYMM"):
            raise
        import sys
        SYMM_FALLBACK = "%s: %s" % (type(e).__name__, str(e).splitlines()[0][:200] if str(e) else "")
        print("runtime: torch symmetric memory unavailable (%s); using CUDA IPC peer mappings" % SYMM_FALLBACK,
              file=sys.stderr, flush=True)
        return _alloc_symmetric_ipc(nbytes, group, device)
    t.zero_()
    return t, [int(p) for p in h.buffer_ptrs], [h]


def multicast_ptr(keep):
    """Multicast (NVLS) address of a symmetric buffer allocated through torch
    symmetric memory (0 when the driver / fabric gives none: one-GPU boxes,
    the CUDA-IPC backend, virtual ranks)."""
    for h in keep or ():
        mc = getattr(h, "multicast_ptr", 0)
        if mc:
            return int(mc)
    return 0


def bind_multicast(st, bits):
    """hand this rank's multicast addresses of the arena, grad
    slots and flag table to the library and select the NVLS kernels (option
    "nvls", bit 0 gathers, bit 1 reduce-scatter).  Returns what was bound;
    the library keeps the unicast kernels for any address that is 0."""
    mc = {k: multicast_ptr(st.peer_keep.get(k)) for k in ("arena", "grad", "flags")}
    if not mc["flags"]:
        mc = {k: 0 for k in mc}
    dc.check(dc.lib.dc_bind_multicast(st.ctx, mc["arena"] if bits & 1 else 0, mc["grad"] if bits & 2 else 0,
                                      mc["flags"]), st.ctx)
    dc.check(dc.lib.dc_set_option(st.ctx, b"nvls", bits), st.ctx)
    st.nvls = {"requested": bits, "ag_multimem": bool(bits & 1 and mc["arena"]),
               "rs_ld_reduce": bool(bits & 2 and mc["grad"])}
    return st.nvls


def create_ranks(table, world, device=0, *, virtual=True, group=None, rank=0, lr=1e-3, beta1=0.9,
                 beta2=0.999, eps=1e-8, seed=0, init=True, host_pinned_bytes=0, spin_ms=None, extra_flags=0,
                 micro_steps=1, defer_states=False):
    """Allocate and dc_init the ranks this process drives: all N virtual ranks,
    or this process's rank when `virtual` is False.  micro_steps > 1: gradient
    accumulation (an fp32 grad-accumulation shard is allocated).  defer_states:
    m / v are not allocated here; bind_host_states() sizes them from the plan
    (host-resident offload, reading D28)."""
    dev = torch.device("cuda", device)
    if spin_ms is None:                      # device flag-wait bound (ms)
        spin_ms = int(os.environ.get("DC_SPIN_MS", "20000"))
    numel, layer_of, init_k = table_arrays(table)
    mops = max_s0_ops(table, micro_steps)
    la = dc.LayoutArgs(world, len(table), dc.i64_array(numel), dc.i32_array(layer_of), mops)
    lay = dc.Layout()
    dc.check(dc.lib.dc_layout_query(C.byref(la), C.byref(lay)))
    mine = list(range(world)) if virtual else [rank]
    ranks = {r: RankState() for r in mine}
    grad_bytes = 2 * lay.grad_slot_bytes
    if virtual:
        for r in mine:
            ranks[r].tensors["grad"] = torch.zeros(grad_bytes, dtype=torch.uint8, device=dev)
            ranks[r].tensors["flags"] = torch.zeros(lay.flag_bytes, dtype=torch.uint8, device=dev)
        grad_ptrs = [ranks[r].tensors["grad"].data_ptr() for r in mine]
        flag_ptrs = [ranks[r].tensors["flags"].data_ptr() for r in mine]
    else:
        g, grad_ptrs, gk = _alloc_symmetric(grad_bytes, group, dev)
        f, flag_ptrs, fk = _alloc_symmetric(lay.flag_bytes, group, dev)
        ranks[rank].tensors["grad"], ranks[rank].tensors["flags"] = g, f
        ranks[rank].peer_keep["grad"], ranks[rank].peer_keep["flags"] = gk, fk
    for r in mine:
        st = ranks[r]
        t = st.tensors
        t["shard"] = torch.empty(lay.shard_elems, dtype=torch.bfloat16, device=dev)
        t["master"] = torch.empty(lay.shard_elems, dtype=torch.float32, device=dev)
        if not defer_states:
            t["m"] = torch.empty(lay.shard_elems, dtype=torch.float32, device=dev)
            t["v"] = torch.empty(lay.shard_elems, dtype=torch.float32, device=dev)
        if micro_steps > 1:
            t["acc"] = torch.empty(lay.shard_elems, dtype=torch.float32, device=dev)
        if host_pinned_bytes:
            t["host"] = torch.empty(host_pinned_bytes, dtype=torch.uint8, pin_memory=True)
        a = dc.InitArgs()
        a.rank, a.world, a.device, a.n_params = r, world, device, len(table)
        st._keep = [dc.i64_array(numel), dc.i32_array(layer_of), dc.f32_array(init_k),
                    dc.u64_array(grad_ptrs), dc.u64_array(flag_ptrs)]
        a.numel, a.layer_of, a.init_k = (C.cast(st._keep[0], dc.p_i64), C.cast(st._keep[1], dc.p_i32),
                                         C.cast(st._keep[2], dc.p_f32))
        a.max_s0_ops = mops
        a.shard_param, a.master = t["shard"].data_ptr(), t["master"].data_ptr()
        a.exp_avg, a.exp_avg_sq = (None, None) if defer_states else (t["m"].data_ptr(), t["v"].data_ptr())
        a.grad_peer_ptrs, a.grad_bytes = C.cast(st._keep[3], dc.p_u64), grad_bytes
        a.flag_peer_ptrs, a.flag_bytes = C.cast(st._keep[4], dc.p_u64), lay.flag_bytes
        a.host_pinned = t["host"].data_ptr() if host_pinned_bytes else None
        a.host_pinned_bytes = host_pinned_bytes
        a.lr, a.beta1, a.beta2, a.eps = lr, beta1, beta2, eps
        a.seed = seed
        a.flags = (dc.DC_INIT_WEIGHTS if init else 0) | (dc.DC_VIRTUAL_RANKS if virtual else 0) | extra_flags | \
            (dc.DC_DEFER_STATES if defer_states else 0)
        a.spin_limit = spin_ms
        a.micro_steps = micro_steps
        a.grad_acc = t["acc"].data_ptr() if micro_steps > 1 else None
        st.micro_steps = micro_steps
        out = C.c_void_p()
        dc.check(dc.lib.dc_init(C.byref(a), C.byref(out)))
        st.ctx = out
        st.rank = r
        st.world = world
        st.layout = lay
        st.device = dev
        # compute, ag, rs, copy.  DC_STREAM_PRIO=compute gives the compute
        # stream the higher priority (rs_adam then fills in behind the GEMMs)
        prio = os.environ.get("DC_STREAM_PRIO", "none")
        st.streams = [torch.cuda.Stream(device=dev, priority=(-1 if (i == 0 and prio == "compute") else 0))
                      for i in range(4 if not (virtual and world >= 8) else 3)]
        if len(st.streams) == 3:
            # 8 virtual ranks share one GPU's 32 hardware connections: with 4+ streams per rank
            # some streams of different ranks share a queue, and a rank's spin-wait kernel can
            # then sit in front of the peer work it waits for (profiles/r02/stalls/); the copy
            # stream (offload only) shares the reduce-scatter stream here, and attach_model
            # keeps the dW GEMMs on the compute stream
            st.streams.append(st.streams[2])
    return ranks


def shard_range(st, p):
    off, S = C.c_int64(), C.c_int64()
    dc.check(dc.lib.dc_shard_range(st.ctx, p, C.byref(off), C.byref(S)), st.ctx)
    return off.value, S.value


def grad_offset(st, p):
    b = C.c_int64()
    dc.check(dc.lib.dc_grad_offset(st.ctx, p, C.byref(b)), st.ctx)
    return b.value


def attach_model(ranks, cfg, xs, targets, checkpoint=False):
    """dc_model_create + bind per rank; xs/targets: dict rank -> bf16 device
    [n, T, H] (n = micro_steps micro-batches; [T, H] when n = 1)."""
    d = dc.ModelDims(cfg.hidden, cfg.ffn, cfg.n_heads, cfg.n_kv, cfg.head_dim, cfg.layers, cfg.tokens,
                     int(checkpoint), int(getattr(cfg, "n_experts", 0)))
    for r, st in ranks.items():
        m = C.c_void_p()
        dc.check(dc.lib.dc_model_create(st.ctx, C.byref(d), C.byref(m)))
        st.model = m
        nb = C.c_uint64()
        dc.check(dc.lib.dc_model_act_bytes(m, C.byref(nb)))
        st.tensors["act"] = torch.empty(nb.value, dtype=torch.uint8, device=st.device)
        st.tensors["x"], st.tensors["t"] = xs[r], targets[r]
        dc.check(dc.lib.dc_model_bind(m, st.tensors["act"].data_ptr(), nb.value, xs[r].data_ptr(),
                                      targets[r].data_ptr()))
        if len(ranks) >= 8:      # virtual ranks: no second GEMM stream (see create_ranks)
            dc.check(dc.lib.dc_model_set_option(m, b"dw_concurrent", 0))
            st.aux_streams = [st.streams[2]]
        elif len(ranks) > 1:
            # virtual ranks: the dW and write-back streams come from torch's stream pool
            # like the rank's other streams (distinct hardware queues), not from
            # cudaStreamCreate inside the library, whose queue is whichever one the
            # process-wide round robin reached — possibly one a peer's spin-wait holds
            st.aux_streams = [torch.cuda.Stream(device=st.device) for _ in range(2)]
        if len(ranks) > 1:
            dc.check(dc.lib.dc_model_set_option(m, b"dw_stream", st.aux_streams[0].cuda_stream), st.ctx)
            dc.check(dc.lib.dc_model_set_option(m, b"wb_stream", st.aux_streams[-1].cuda_stream), st.ctx)


def bind(ranks, sched_by_rank, group=None):
    """Allocate the gather arena at the planned capacity and dc_bind_schedule
    on every rank (all ranks quiescent)."""
    any_st = next(iter(ranks.values()))
    cap = max(1, int(dc.lib.dc_schedule_capacity(next(iter(sched_by_rank.values())))))
    if any_st.world == 1:
        ptrs = {r: [0] for r in ranks}
    elif group is None:   # virtual ranks
        for r, st in ranks.items():
            st.tensors["arena"] = torch.empty(cap, dtype=torch.uint8, device=st.device)
        allp = [ranks[r].tensors["arena"].data_ptr() for r in sorted(ranks)]
        ptrs = {r: allp for r in ranks}
    else:
        st = any_st
        # drop the previous arena's peer mappings before mapping the new one
        st.peer_keep.pop("arena", None)
        st.tensors.pop("arena", None)
        t, allp, keep = _alloc_symmetric(cap, group, st.device)
        st.tensors["arena"] = t
        st.peer_keep["arena"] = keep
        ptrs = {st.rank: allp}
    torch.cuda.synchronize()
    for r, st in ranks.items():
        st.sched = sched_by_rank[r]
        arr = dc.u64_array(ptrs[r])
        st._arena_keep = arr
        dc.check(dc.lib.dc_bind_schedule(st.ctx, st.sched, C.cast(arr, dc.p_u64), cap,
                                         st.streams[0].cuda_stream), st.ctx)
    torch.cuda.synchronize()
    nvls = int(os.environ.get("DC_NVLS", "0"))
    if group is not None and nvls:
        bind_multicast(any_st, nvls)
    if group is not None:
        # dc_bind_schedule zeroes this rank's flag table; no rank may start a
        # step (whose first action posts ready flags into its peers' tables)
        # before every peer's zeroing is done
        import torch.distributed as dist
        dist.barrier(group=group)


def max_reduce_profile(prof, group, device="cpu"):
    """Element-wise MAX of (p_mem, transient, dur_us) over the ranks of `group`
    (reading D12: every rank must plan from the same profile, or the symmetric
    arena and the flag protocol diverge).  Works over gloo (cpu) and nccl."""
    import torch.distributed as dist
    vals = torch.tensor([[o["p_mem"], o["transient"], o["dur_us"]] for o in prof["ops"]], dtype=torch.int64,
                        device=device)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX, group=group)
    out = json.loads(json.dumps(prof))
    for o, v in zip(out["ops"], vals.tolist()):
        o["p_mem"], o["transient"], o["dur_us"] = v
    if out.get("tc"):
        tcv = torch.tensor([t[1] for t in out["tc"]], dtype=torch.int64, device=device)
        dist.all_reduce(tcv, op=dist.ReduceOp.MAX, group=group)
        out["tc"] = [[t[0], int(v)] for t, v in zip(out["tc"], tcv.tolist())]
    return out


def plan_digest(sched_json):
    import hashlib
    return hashlib.sha256(sched_json.encode()).hexdigest()


def offload_fragments(st, max_fragment_bytes):
    """dc_offload_fragments -> planner fragment records {id, layer, bytes}.
    The full records (state, element offset and count, pinned host byte
    offset: fragments are packed in id order) are kept on the rank state."""
    n = C.c_int32(0)
    dc.check(dc.lib.dc_offload_fragments(st.ctx, max_fragment_bytes, None, C.byref(n)), st.ctx)
    arr = (dc.Fragment * n.value)()
    dc.check(dc.lib.dc_offload_fragments(st.ctx, max_fragment_bytes, arr, C.byref(n)), st.ctx)
    st.frags, host_off = [], 0
    for f in arr:
        st.frags.append(dict(layer=f.layer, state=f.state, off=f.offset_elems, elems=f.elems, host_off=host_off))
        host_off += f.elems * 4
    return [dict(id=i, layer=f.layer, bytes=f.elems * 4) for i, f in enumerate(arr)]


def layer_state_bytes(table, world):
    """Bytes of the largest layer's m (or v) shard: dc_offload_fragments with
    this maximum gives whole (layer, state) fragments (host-resident mode)."""
    per = {}
    for p in table:
        per[p.layer] = per.get(p.layer, 0) + -(-p.numel // (8 * world)) * 8
    return 4 * max(per.values())


def bind_host_states(ranks, alloc_host=False, extra_slots=0):
    """After bind(): size m / v to the elements the plan keeps on the device,
    allocate the reload ring pool and dc_model_bind_host_states (states reset
    to zero; reading D28).  alloc_host: allocate the pinned host slots now, at
    the size the offloaded fragments need (else dc_init's host_pinned buffer
    is used).  Returns {rank: (m_first, v_first, pool_bytes, host_bytes)}."""
    out = {}
    for r, st in ranks.items():
        mf, vf, pb, hb = C.c_int64(), C.c_int64(), C.c_uint64(), C.c_uint64()
        dc.check(dc.lib.dc_model_host_states_query(st.model, C.byref(mf), C.byref(vf), C.byref(pb), C.byref(hb)),
                 st.ctx)
        E = st.layout.shard_elems
        t = st.tensors
        t["m"] = torch.empty(max(E - mf.value, 4), dtype=torch.float32, device=st.device)
        t["v"] = torch.empty(max(E - vf.value, 4), dtype=torch.float32, device=st.device)
        extra = 0
        if pb.value and extra_slots:      # slot = the largest offloaded fragment, 256 B aligned
            offl = [f for f in st.frags if f["off"] < (mf.value if f["state"] == 0 else vf.value)]
            extra = extra_slots * max(-(-f["elems"] // 64) * 64 * 4 for f in offl)
        pbytes = pb.value + extra
        t["pool"] = torch.empty(max(pbytes, 256), dtype=torch.uint8, device=st.device)
        host, hbytes = None, 0
        if alloc_host:
            t["host"] = torch.empty(max(hb.value, 256), dtype=torch.uint8, pin_memory=True)
            host, hbytes = t["host"].data_ptr(), t["host"].numel()
        dc.check(dc.lib.dc_model_bind_host_states(st.model, t["m"].data_ptr(), t["v"].data_ptr(),
                                                  t["pool"].data_ptr(), pbytes, host, hbytes), st.ctx)
        st.host_states = (mf.value, vf.value, pbytes, hb.value)
        out[r] = st.host_states
    return out


def full_states(st):
    """(m, v) fp32 on the CPU over all shard elements: the device-resident part
    plus the offloaded fragments' pinned host copies (tests / diagnostics)."""
    if not getattr(st, "host_states", None):
        return st.tensors["m"].cpu(), st.tensors["v"].cpu()
    mf, vf = st.host_states[:2]
    E = st.layout.shard_elems
    host = st.tensors["host"].view(torch.float32)
    out = []
    for state, first, dev in ((0, mf, st.tensors["m"]), (1, vf, st.tensors["v"])):
        full = torch.empty(E, dtype=torch.float32)
        full[first:] = dev[:E - first].cpu()
        for f in st.frags:
            if f["state"] == state and f["off"] < first:
                h = f["host_off"] // 4
                full[f["off"]:f["off"] + f["elems"]] = host[h:h + f["elems"]]
        out.append(full)
    return tuple(out)


def profile_json(st, tc=None, frags=None):
    prof = json.loads(dc.model_profile_json(st.model))
    prof["tc"] = tc if tc is not None else [[0, 0], [1 << 40, 0]]
    prof["frags"] = frags or []
    return prof


def run_parallel(ranks, fn):
    """Run fn(rank_state) for every rank, each in its own thread (virtual ranks
    spin on each other's flags, so their host calls must interleave)."""
    if len(ranks) == 1:
        st = next(iter(ranks.values()))
        fn(st)
        return
    errs = []

    def wrap(st):
        try:
            torch.cuda.set_device(st.device)
            fn(st)
        except BaseException as e:   # noqa: BLE001 - re-raised below
            errs.append(e)

    th = [threading.Thread(target=wrap, args=(st,)) for st in ranks.values()]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]


def step(ranks, t, profile=False):
    """One dc_model_step per rank (profile: False/0, True/1 = record+read,
    2 = record only).  Several virtual ranks in this process: returns once
    their step has finished on the device, so the spin-waits of one set of
    virtual ranks never share hardware queues with another set's work that
    a later call enqueues (a wait at a queue's head blocks everything behind
    it: profiles/r02/stalls/).  One rank per process: asynchronous."""
    mode = int(profile) if not isinstance(profile, bool) else (1 if profile else 0)

    def one(st):
        dc.check(dc.lib.dc_model_step(st.model, t, mode, *st.stream_handles()), st.ctx)
    run_parallel(ranks, one)
    if len(ranks) > 1:
        torch.cuda.synchronize()


def poll(ranks):
    """Raise if any rank's device flag wait timed out (sticky error word); the
    message carries every failing rank's record (which flag each one waited
    on), so a cross-rank stall shows both ends."""
    errs = []
    for st in ranks.values():
        status = dc.lib.dc_poll(st.ctx)
        if status != dc.DC_OK:
            errs.append((status, dc.last_error(st.ctx)))
    if errs:
        raise dc.DCError(errs[0][0], " | ".join(m for _, m in errs))


def loss_ptr(st):
    p = dc.p_f32()
    dc.check(dc.lib.dc_model_loss_ptr(st.model, C.byref(p)))
    return C.cast(p, C.c_void_p).value


class _CAI:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


_TYPESTR = {torch.float32: "<f4", torch.uint8: "|u1", torch.int16: "<i2", torch.uint32: "<u4",
            torch.bfloat16: "<i2"}


def view(ptr, n, dtype, device="cuda"):
    """Zero-copy torch view (n elements) of library-addressed device memory,
    e.g. dc_tensor_ptr / dc_grad_slot results (tests and diagnostics only)."""
    t = torch.as_tensor(_CAI(int(ptr), n, _TYPESTR[dtype]), device=device)
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t
