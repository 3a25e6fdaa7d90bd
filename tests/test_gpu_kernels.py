"""GPU parity of the individual hot-path kernels against the oracle, through
the C ABI (tests run on a B200 under gpurun: pytest -m gpu).

* init:    dc_init's on-device generator == oracle shard_of(values)  (bit-exact)
* gemm:    tcgen05 GEMM, all operand layouts / segments / ragged tails / residual
           vs an fp64 matmul of the same bf16 inputs (bf16 output tolerance)
* rs_adam: reduce-scatter + 1/N + Adam in DC_VIRTUAL_RANKS mode, N in {1,2,4},
           two steps, vs oracle.numerics.rs_adam_shard (bit-exact; <= 1e-5 bar)
* ag_push: every gather of a planned schedule, N in {2,4,8} virtual ranks,
           vs oracle all_gather (bit-exact, including padding)
"""
import ctypes as C
import json
import os

import numpy as np
import pytest
import torch

import synth
from oracle import numerics as nx
from oracle import step as ost
from tests import sched_util as su
from tests.gpu_util import bf16_tensor, seeded, to_np

pytestmark = pytest.mark.gpu

dc = pytest.importorskip("paper_2504_09983_b200.dc")
from paper_2504_09983_b200 import runtime as rt  # noqa: E402


# ------------------------------------------------------------------ init
def test_init_bitexact():
    cfg = synth.small_llama(layers=2)
    table = synth.llama_param_table(cfg)
    full = ost.init_full_params(table)
    for world in (1, 2):
        ranks = rt.create_ranks(table, world, seed=synth.SEED_WEIGHTS)
        torch.cuda.synchronize()
        for r, st in ranks.items():
            sh = st.tensors["shard"].view(torch.int16).cpu().numpy().view(np.uint16)
            ms = st.tensors["master"].cpu().numpy()
            for i, p in enumerate(table):
                off, S = rt.shard_range(st, i)
                ref = nx.shard_of(full[i], world, r)
                assert ms[off:off + S].tobytes() == ref.tobytes(), (r, p.name)
                assert np.array_equal(sh[off:off + S], nx.bf16_bits(ref)), (r, p.name)
            assert not st.tensors["m"].any() and not st.tensors["v"].any()


# ------------------------------------------------------------------ GEMM
_WS = {}


def _workspace():
    """Caller-owned stream-K workspace (dc_gemm_args.workspace), zero-filled."""
    if "ws" not in _WS:
        _WS["ws"] = torch.zeros(int(dc.lib.dc_gemm_workspace_bytes()), dtype=torch.uint8, device="cuda")
    return _WS["ws"]


def _gemm(M, N, K, A, lda, a_mn, Bs, ldbs, ends, b_mn, split_k, Cm, ldc, R=None, ldr=0, sms=0, kernel=0, sk=0,
          group_m=0):
    g = dc.GemmArgs()
    g.M, g.N, g.K = M, N, K
    g.A, g.lda, g.a_mn_major = A.data_ptr(), lda, a_mn
    g.n_bseg = len(Bs)
    for i, (b, l, e) in enumerate(zip(Bs, ldbs, ends)):
        g.B[i], g.ldb[i], g.bseg_end[i] = b.data_ptr(), l, e
    g.b_mn_major, g.b_split_k = b_mn, split_k
    g.C, g.ldc = Cm.data_ptr(), ldc
    g.R, g.ldr = (R.data_ptr() if R is not None else None), ldr
    g.num_sms = sms
    # kernel 1: one-CTA tiles; 2: CTA pairs 256 x 256; 3: CTA pairs 256 x 128
    os.environ["DC_GEMM_BN"] = "128" if kernel == 3 else "256"
    g.kernel = 2 if kernel == 3 else kernel
    g.stream_k = sk
    if sk:
        ws = _workspace()
        g.workspace, g.workspace_bytes = ws.data_ptr(), ws.numel()
    g.tile_group_m = group_m
    dc.check(dc.lib.dc_gemm(C.byref(g), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()


def _check(Cm, ref, absref, name):
    got = to_np(Cm)
    err = np.abs(got - ref)
    tol = 2.0 ** -8 * np.abs(ref) + 2.0 ** -18 * absref + 1e-30
    bad = err > tol
    assert not bad.any(), "%s: %d bad, max err %g" % (name, bad.sum(), err.max())


def _mat(seed, r, c):
    a = nx.rne_bf16(seeded(seed, 0, r * c)).reshape(r, c)
    return a, bf16_tensor(a)


KERNELS = pytest.mark.parametrize("kernel", [1, 2, 3], ids=["cta1", "pair256", "pair128"])


@KERNELS
@pytest.mark.parametrize("M,N,K,sms", [(256, 512, 512, 0), (200, 264, 200, 0), (1024, 2048, 1024, 8),
                                       (130, 8, 64, 0), (600, 776, 136, 6)])
def test_gemm_forward_kmajor(M, N, K, sms, kernel):
    a, A = _mat(11, M, K)
    b, B = _mat(12, N, K)
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, K, A, K, 0, [B], [K], [0], 0, 0, Cm, N, sms=sms, kernel=kernel)
    _check(Cm, a @ b.T, np.abs(a) @ np.abs(b).T, "fwd")


@KERNELS
def test_gemm_nsplit_segments_and_residual(kernel):
    M, K = 384, 320
    Ns = [256, 256, 512]
    a, A = _mat(21, M, K)
    bs = [_mat(22 + i, n, K) for i, n in enumerate(Ns)]
    r, R = _mat(30, M, sum(Ns))
    Cm = torch.empty(M, sum(Ns), dtype=torch.bfloat16, device="cuda")
    _gemm(M, sum(Ns), K, A, K, 0, [x[1] for x in bs], [K] * 3, [1, 2, 4], 0, 0, Cm, sum(Ns), R=R, ldr=sum(Ns), kernel=kernel)
    bcat = np.concatenate([x[0] for x in bs])
    ref = (a @ bcat.T) + r
    _check(Cm, ref, np.abs(a) @ np.abs(bcat).T + np.abs(r), "nsplit+res")


@KERNELS
def test_gemm_ksplit_mn_major_b(kernel):
    """dX = dY W with W split along K (q|k|v): B stored [K_s][N] (N contiguous)."""
    M, N = 256, 512
    Ks = [128, 64, 192]
    a, A = _mat(41, M, sum(Ks))
    ws = [_mat(42 + i, k, N) for i, k in enumerate(Ks)]
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, sum(Ks), A, sum(Ks), 0, [w[1] for w in ws], [N] * 3, [2, 3, 6], 1, 1, Cm, N, kernel=kernel)
    wcat = np.concatenate([w[0] for w in ws])
    _check(Cm, a @ wcat, np.abs(a) @ np.abs(wcat), "ksplit")


def _silu(z):
    return z / (1.0 + np.exp(-z))


@pytest.mark.parametrize("M,F,K", [(256, 256, 192), (200, 384, 136), (600, 512, 64)])
def test_gemm_glu_epilogues(M, F, K):
    """Epilogue 2 (gate|up GEMM -> gu + SiLU(g) * u) and 3 (dact GEMM ->
    d(gate | up) from gu): gu bit-identical to the plain segmented GEMM, act /
    d(gate) / d(up) vs fp64 of the same bf16 operands; ragged M."""
    x, X = _mat(81, M, K)
    wg, WG = _mat(82, F, K)
    wu, WU = _mat(83, F, K)
    plain = torch.empty(M, 2 * F, dtype=torch.bfloat16, device="cuda")
    _gemm(M, 2 * F, K, X, K, 0, [WG, WU], [K, K], [F // 256 if F % 256 == 0 else 0, 2 * F // 256], 0, 0, plain, 2 * F,
          kernel=2) if F % 256 == 0 else None
    gu = torch.full((M, 2 * F), float("nan"), dtype=torch.bfloat16, device="cuda")
    act = torch.full((M, F), float("nan"), dtype=torch.bfloat16, device="cuda")
    g = dc.GemmArgs()
    g.M, g.N, g.K = M, F, K
    g.A, g.lda, g.a_mn_major = X.data_ptr(), K, 0
    g.n_bseg = 2
    g.B[0], g.B[1], g.ldb[0], g.ldb[1] = WG.data_ptr(), WU.data_ptr(), K, K
    g.C, g.ldc, g.kernel = gu.data_ptr(), 2 * F, 2
    g.epilogue, g.aux, g.ld_aux, g.glu_off = 2, act.data_ptr(), F, F
    os.environ["DC_GEMM_BN"] = "256"
    dc.check(dc.lib.dc_gemm(C.byref(g), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ref = np.concatenate([x @ wg.T, x @ wu.T], axis=1)
    _check(gu, ref, np.abs(x) @ np.abs(np.concatenate([wg, wu]).T), "glu fwd gu")
    if F % 256 == 0:
        assert torch.equal(gu.view(torch.int16), plain.view(torch.int16))
    gun = to_np(gu)
    a_ref = _silu(gun[:, :F]) * gun[:, F:]
    _check(act, a_ref, np.abs(a_ref), "glu fwd act")
    # backward: dact = dY Wd (Wd stored [K rows][F], MN-major), epilogue 3
    dy, DY = _mat(84, M, K)
    wd, WD = _mat(85, K, F)
    dgu = torch.full((M, 2 * F), float("nan"), dtype=torch.bfloat16, device="cuda")
    g = dc.GemmArgs()
    g.M, g.N, g.K = M, F, K
    g.A, g.lda, g.a_mn_major = DY.data_ptr(), K, 0
    g.n_bseg = 1
    g.B[0], g.ldb[0], g.bseg_end[0] = WD.data_ptr(), F, F // 256 if F >= 256 else 1
    g.b_mn_major = 1
    g.C, g.ldc, g.kernel = dgu.data_ptr(), 2 * F, 2
    g.epilogue, g.aux, g.ld_aux, g.glu_off = 3, gu.data_ptr(), 2 * F, F
    dc.check(dc.lib.dc_gemm(C.byref(g), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    da = nx.rne_bf16(dy @ wd)
    gg, uu = gun[:, :F], gun[:, F:]
    s = 1.0 / (1.0 + np.exp(-gg))
    dg_ref, du_ref = da * uu * s * (1 + gg * (1 - s)), da * gg * s
    got = to_np(dgu)
    for name, gv, rv in (("d(gate)", got[:, :F], dg_ref), ("d(up)", got[:, F:], du_ref)):
        err = np.abs(gv - rv)
        assert (err <= 2.0 ** -7 * np.abs(rv) + 1e-6 * np.abs(rv).max()).all(), (name, err.max())
    # refused combinations
    g.R = gu.data_ptr()
    assert dc.lib.dc_gemm(C.byref(g), torch.cuda.current_stream().cuda_stream) == dc.DC_EINVAL


@KERNELS
@pytest.mark.parametrize("M,N,K,sms", [(384, 512, 296, 0), (512, 256, 1024, 4), (256, 256, 64, 0)])
def test_gemm_dw_both_mn_major(M, N, K, sms, kernel):
    """dW = dY^T X: A stored [K][M], B stored [K][N]; A slice with lda > M."""
    dy, DY = _mat(51, K, M + 64)          # use columns [64, 64+M) via pointer offset
    x, X = _mat(52, K, N)
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, K, DY[:, 64:], M + 64, 1, [X], [N], [0], 1, 0, Cm, N, sms=sms, kernel=kernel)
    ref = dy[:, 64:].T @ x
    _check(Cm, ref, np.abs(dy[:, 64:]).T @ np.abs(x), "dW")


def test_gemm_rejects_bad_shapes():
    A = torch.empty(8, 8, dtype=torch.bfloat16, device="cuda")
    g = dc.GemmArgs()
    g.M, g.N, g.K, g.n_bseg = 8, 7, 8, 1
    g.A = g.B[0] = g.C = A.data_ptr()
    assert dc.lib.dc_gemm(C.byref(g), None) == dc.DC_EINVAL


# stream-K tails: with `sms` pairs' worth of SMs and a tile count that is not a
# multiple of the pair count, the last [P, 2P) tiles are split into P equal
# k-ranges; split tiles add the head's fp32 partial in the tail's epilogue.
# (stream-K needs k_blocks >= 128, i.e. K > 8128)
SK_CASES = pytest.mark.parametrize("M,N,K,sms", [(768, 1280, 8192, 8), (640, 1024, 8200, 6), (2048, 2560, 8192, 0)])


@pytest.mark.parametrize("kernel", [2, 3], ids=["pair256", "pair128"])
@SK_CASES
def test_gemm_stream_k_forward_residual(M, N, K, sms, kernel):
    a, A = _mat(61, M, K)
    b, B = _mat(62, N, K)
    r, R = _mat(63, M, N)
    outs = []
    for sk in (1, 1, 0):
        Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        _gemm(M, N, K, A, K, 0, [B], [K], [0], 0, 0, Cm, N, R=R, ldr=N, sms=sms, kernel=kernel, sk=sk)
        outs.append(Cm)
    _check(outs[0], a @ b.T + r, np.abs(a) @ np.abs(b).T + np.abs(r), "sk fwd")
    assert torch.equal(outs[0], outs[1])                  # deterministic split and sum order
    _check(outs[2], a @ b.T + r, np.abs(a) @ np.abs(b).T + np.abs(r), "dp fwd")


@SK_CASES
def test_gemm_stream_k_dx_dw(M, N, K, sms):
    # dX layout with B split along K into two segments
    a, A = _mat(71, M, K)
    k1 = (K // 2) // 64 * 64
    w1, W1 = _mat(72, k1, N)
    w2, W2 = _mat(73, K - k1, N)
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, K, A, K, 0, [W1, W2], [N, N], [k1 // 64, -(-K // 64)], 1, 1, Cm, N, sms=sms, kernel=2, sk=1)
    wcat = np.concatenate([w1, w2])
    _check(Cm, a @ wcat, np.abs(a) @ np.abs(wcat), "sk dx")
    # dW layout: A stored [K][M], B stored [K][N]
    dy, DY = _mat(74, K, M)
    x, X = _mat(75, K, N)
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, K, DY, M, 1, [X], [N], [0], 1, 0, Cm, N, sms=sms, kernel=2, sk=1)
    _check(Cm, dy.T @ x, np.abs(dy).T @ np.abs(x), "sk dw")


# tile order of the persistent pair kernel: groups of g m-tiles, including a
# partial last group (m_tiles % g != 0) and its combination with a stream-K
# tail; the output must not depend on the order (each tile is computed once)
@pytest.mark.parametrize("group_m", [-1, 2, 3, 8])
@pytest.mark.parametrize("sk", [0, 1])
def test_gemm_tile_groups_partial(group_m, sk):
    M, N, K, sms = 5 * 256, 256, 8256 if sk else 512, 6
    a, A = _mat(81, M, K)
    b, B = _mat(82, N, K)
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, K, A, K, 0, [B], [K], [0], 0, 0, Cm, N, sms=sms, kernel=2, sk=sk, group_m=group_m)
    _check(Cm, a @ b.T, np.abs(a) @ np.abs(b).T, "groups g=%d sk=%d" % (group_m, sk))
    ref = torch.empty_like(Cm)
    _gemm(M, N, K, A, K, 0, [B], [K], [0], 0, 0, ref, N, sms=sms, kernel=2, sk=0, group_m=-1)
    assert torch.equal(Cm, ref) if not sk else True      # data-parallel tiles: same k order


def test_gemm_stream_k_needs_workspace():
    """stream_k without a workspace runs data-parallel (no library allocation);
    a too-small workspace is DC_EINVAL."""
    M, N, K = 768, 1280, 8192
    a, A = _mat(91, M, K)
    b, B = _mat(92, N, K)
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    g = dc.GemmArgs()
    g.M, g.N, g.K = M, N, K
    g.A, g.lda = A.data_ptr(), K
    g.n_bseg, g.B[0], g.ldb[0] = 1, B.data_ptr(), K
    g.C, g.ldc = Cm.data_ptr(), N
    g.num_sms, g.kernel, g.stream_k = 8, 2, 1
    dc.check(dc.lib.dc_gemm(C.byref(g), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    _check(Cm, a @ b.T, np.abs(a) @ np.abs(b).T, "sk without workspace")
    small = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    g.workspace, g.workspace_bytes = small.data_ptr(), small.numel()
    assert dc.lib.dc_gemm(C.byref(g), torch.cuda.current_stream().cuda_stream) == dc.DC_EINVAL


# ------------------------------------------------------------------ RS + Adam
def _grads(world, table, S, q, step, micro=0):
    out = []
    for i, p in enumerate(table):
        g = nx.rne_bf16(seeded(500 + 10 * step + q + 4096 * micro, i, p.numel, std=0.01))
        out.append(np.concatenate([g, np.zeros(world * S[i] - p.numel, np.float32)]))
    return out


def _bits_equal(got, ref, what):
    rel = np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), 1e-30)
    assert rel.max() <= 1e-5, (what, rel.max())
    assert got.tobytes() == ref.tobytes(), (what, "not bit-exact")


def _ragged_table():
    """Edge-case parameter sizes: smaller than one 16 B shard vector per rank
    (1, 7), odd (13, 4099, 65537) and a 1 MiB tensor; two layers.  Params 0
    and 3 start at zero, so after step 1 their fp32 master IS the Adam update
    (every bit visible: a 1-ulp error in sqrt(v)/c + eps or in the final
    division, absorbed when added to a weight of ~0.02, fails here)."""
    sizes = [(0, 1), (0, 7), (0, 4099), (0, 1 << 19), (1, 13), (1, 65537), (1, 24)]
    k = float(synth.std_to_k(0.02))
    return [synth.ParamSpec(id=i, layer=l, name="p%d" % i, shape=(n,), k=(0.0 if i in (0, 3) else k), dtype="bf16")
            for i, (l, n) in enumerate(sizes)]


RS_BULK = pytest.mark.parametrize("bulk", [0, 1], ids=["ldg", "bulk"])


@RS_BULK
@pytest.mark.parametrize("world,n,ragged", [(1, 1, False), (2, 1, False), (4, 1, False), (1, 2, False),
                                            (2, 3, False), (4, 2, False), (3, 1, True), (8, 2, True)])
def test_rs_adam_virtual_ranks(world, n, ragged, bulk):
    """rs_adam (n = 1) and its gradient-accumulation modes (n > 1: acc = rs,
    acc += rs, then Adam on (acc + rs) / (N n)) vs the oracle, bit-exact,
    two optimizer steps, the accumulator checked after every micro-step.
    Ragged: tiny / odd tensors (mostly padding at N = 8) and N = 3 (1/N inexact).
    bulk: the bulk-copy pipelined kernel (update / final modes) — chunk tails
    (S % 2048), members smaller than one chunk, more CTAs than chunks."""
    cfg = synth.small_llama(layers=2)
    table = _ragged_table() if ragged else synth.llama_param_table(cfg)
    lr = 1e-3
    ranks = rt.create_ranks(table, world, lr=lr, micro_steps=n)
    for st in ranks.values():
        dc.check(dc.lib.dc_set_option(st.ctx, b"rs_bulk", bulk), st.ctx)
    S = [nx.shard_len(p.numel, world) for p in table]
    full = ost.init_full_params(table)
    o_master = [[nx.shard_of(full[i], world, r) for i in range(len(table))] for r in range(world)]
    o_m = [[np.zeros(S[i], np.float32) for i in range(len(table))] for r in range(world)]
    o_v = [[np.zeros(S[i], np.float32) for i in range(len(table))] for r in range(world)]
    for step in (1, 2):
        o_acc = [[None] * len(table) for _ in range(world)]
        for mu in range(n):
            grads = {q: _grads(world, table, S, q, step, mu) for q in range(world)}

            def work(st):
                cs, rs = st.streams[0], st.streams[2]
                for layer in (1, 0):
                    dc.check(dc.lib.dc_grad_slot_acquire(st.ctx, layer, cs.cuda_stream), st.ctx)
                    slot = C.c_void_p()
                    dc.check(dc.lib.dc_grad_slot(st.ctx, layer, C.byref(slot)), st.ctx)
                    with torch.cuda.stream(cs):
                        for i, p in enumerate(table):
                            if p.layer != layer:
                                continue
                            v = rt.view(slot.value + rt.grad_offset(st, i), world * S[i], torch.bfloat16)
                            v.copy_(bf16_tensor(grads[st.rank][i]))
                    dc.check(dc.lib.dc_grad_slot_publish(st.ctx, layer, cs.cuda_stream), st.ctx)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    rs.wait_event(ev)                    # local order, as the executor does
                    dc.check(dc.lib.dc_reduce_scatter_step(st.ctx, layer, step, mu, rs.cuda_stream), st.ctx)
                torch.cuda.synchronize()

            rt.run_parallel(ranks, work)
            rt.poll(ranks)
            for r, st in ranks.items():
                for i, p in enumerate(table):
                    gq = [grads[q][i] for q in range(world)]
                    off, sz = rt.shard_range(st, i)
                    if mu < n - 1:
                        o_acc[r][i] = nx.accumulate(o_acc[r][i], nx.reduce_scatter(gq, world, r))
                        _bits_equal(st.tensors["acc"][off:off + sz].cpu().numpy(), o_acc[r][i], (r, p.name, mu))
                        continue
                    mst, m1, v1, shb = nx.rs_adam_shard(gq, o_master[r][i], o_m[r][i], o_v[r][i], world, r,
                                                        step, lr, acc=o_acc[r][i], micro_steps=n)
                    o_master[r][i], o_m[r][i], o_v[r][i] = mst, m1, v1
        for r, st in ranks.items():
            ms, mm, vv = (st.tensors[k].cpu().numpy() for k in ("master", "m", "v"))
            sh = st.tensors["shard"].view(torch.int16).cpu().numpy().view(np.uint16)
            for i, p in enumerate(table):
                off, sz = rt.shard_range(st, i)
                for k, got, ref in (("master", ms, o_master), ("m", mm, o_m), ("v", vv, o_v)):
                    _bits_equal(got[off:off + sz], ref[r][i], (r, p.name, k, step))
                assert np.array_equal(sh[off:off + sz], nx.bf16_bits(o_master[r][i]))


@RS_BULK
@pytest.mark.parametrize("world,step", [(1, 7), (2, 1000)])
def test_rs_adam_random_state(world, step, bulk):
    """rs_adam on arbitrary optimizer states (random master / m / v, v >= 0
    spanning 12 decades) at a later step t: every rounding of Adam's update —
    the sqrt, both divisions, eps — hits general operands, not the
    near-exact quotients of step 1 from a zero state (where sqrt(v)/c is
    |g| almost exactly).  Bit-exact against the oracle."""
    table = _ragged_table()
    lr = 1e-3
    ranks = rt.create_ranks(table, world, lr=lr)
    for st in ranks.values():
        dc.check(dc.lib.dc_set_option(st.ctx, b"rs_bulk", bulk), st.ctx)
    S = [nx.shard_len(p.numel, world) for p in table]
    rng = np.random.default_rng(11 + world)
    states = {}
    for r, st in ranks.items():
        n = st.tensors["master"].numel()
        ms = rng.normal(0.0, 0.02, n).astype(np.float32)
        mm = rng.normal(0.0, 1e-3, n).astype(np.float32)
        vv = (10.0 ** rng.uniform(-14, -2, n)).astype(np.float32)
        for k, a in (("master", ms), ("m", mm), ("v", vv)):
            st.tensors[k].copy_(torch.from_numpy(a))
        states[r] = (ms, mm, vv)
    grads = {q: _grads(world, table, S, q, step) for q in range(world)}

    def work(st):
        cs, rs = st.streams[0], st.streams[2]
        for layer in (1, 0):
            dc.check(dc.lib.dc_grad_slot_acquire(st.ctx, layer, cs.cuda_stream), st.ctx)
            slot = C.c_void_p()
            dc.check(dc.lib.dc_grad_slot(st.ctx, layer, C.byref(slot)), st.ctx)
            with torch.cuda.stream(cs):
                for i, p in enumerate(table):
                    if p.layer == layer:
                        v = rt.view(slot.value + rt.grad_offset(st, i), world * S[i], torch.bfloat16)
                        v.copy_(bf16_tensor(grads[st.rank][i]))
            dc.check(dc.lib.dc_grad_slot_publish(st.ctx, layer, cs.cuda_stream), st.ctx)
            ev = torch.cuda.Event()
            ev.record(cs)
            rs.wait_event(ev)
            dc.check(dc.lib.dc_reduce_scatter_step(st.ctx, layer, step, 0, rs.cuda_stream), st.ctx)
        torch.cuda.synchronize()

    rt.run_parallel(ranks, work)
    rt.poll(ranks)
    for r, st in ranks.items():
        ms0, mm0, vv0 = states[r]
        got = {k: st.tensors[k].cpu().numpy() for k in ("master", "m", "v")}
        sh = st.tensors["shard"].view(torch.int16).cpu().numpy().view(np.uint16)
        for i, p in enumerate(table):
            off, sz = rt.shard_range(st, i)
            sl = slice(off, off + sz)
            ref = nx.rs_adam_shard([grads[q][i] for q in range(world)], ms0[sl], mm0[sl], vv0[sl], world, r, step, lr)
            for k, refk in zip(("master", "m", "v"), ref[:3]):
                _bits_equal(got[k][sl], refk, (r, p.name, k))
            assert np.array_equal(sh[sl], nx.bf16_bits(ref[0])), (r, p.name)


def test_rs_micro_out_of_range():
    cfg = synth.small_llama(layers=1)
    table = synth.llama_param_table(cfg)
    st = rt.create_ranks(table, 1, micro_steps=2)[0]
    cs = st.streams[0]
    dc.check(dc.lib.dc_grad_slot_acquire(st.ctx, 0, cs.cuda_stream), st.ctx)
    assert dc.lib.dc_reduce_scatter_step(st.ctx, 0, 1, 2, cs.cuda_stream) == dc.DC_EINVAL
    assert dc.lib.dc_reduce_scatter_step(st.ctx, 0, 1, -1, cs.cuda_stream) == dc.DC_EINVAL


# ------------------------------------------------------------------ all-gather
def _ops(sched):
    return json.loads(dc.schedule_json(sched))["ops"]


@pytest.mark.parametrize("world,mode", [(3, "sm"), (8, "sm"), (8, "ce"), (3, "bulk"), (8, "bulk"), (8, "chunked")])
def test_ag_ragged_virtual_ranks(world, mode):
    """Gathers of ragged tensors (1 .. 2^19 elements, padded shards) through a
    planned schedule without a model: every gathered buffer == the padded
    concatenation of the shards, bit for bit; SM push (16-byte stores), copy
    engines, bulk-copy pipeline (option ag_bulk) and chunked pushes (fused_ag)."""
    table = _ragged_table()
    ranks = rt.create_ranks(table, world)
    for st in ranks.values():
        dc.check(dc.lib.dc_set_option(st.ctx, b"ag_copy_engine", int(mode == "ce")), st.ctx)
        dc.check(dc.lib.dc_set_option(st.ctx, b"ag_bulk", int(mode == "bulk")), st.ctx)
        dc.check(dc.lib.dc_set_option(st.ctx, b"fused_ag", int(mode == "chunked")), st.ctx)
    B = {p.id: nx.shard_len(p.numel, world) * world * 2 for p in table}
    comp = [("f%d" % p.id, "compute", "fwd", 0, p.layer, [p.id]) for p in table]
    comp += [("b%d" % p.id, "compute", "bwd", 0, p.layer, [p.id]) for p in reversed(table)]
    comp += [("end", "compute", "bwd", 0, 0, [])]              # a profile ends with a compute-like op
    prof = su.make_profile(comp, B, lambda o: 0, tc=[[4096, 10], [1 << 20, 20], [1 << 26, 400]])
    sched = dc.plan(json.dumps(prof), 1 << 40, M_prefetch=1 << 22,
                    passes=dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH, strict=True)
    rt.bind(ranks, {r: sched for r in ranks})
    full = ost.init_full_params(table)
    for st in ranks.values():
        dc.check(dc.lib.dc_step_begin(st.ctx, 1, st.streams[0].cuda_stream), st.ctx)
    checked = []
    for o in _ops(sched):
        if o["kind"] == "ag":
            for st in ranks.values():
                dc.check(dc.lib.dc_gather(st.ctx, o["id"], st.streams[1].cuda_stream, None), st.ctx)
            torch.cuda.synchronize()
            for st in ranks.values():
                for p in o["members"]:
                    ptr = C.c_void_p()
                    dc.check(dc.lib.dc_tensor_ptr(st.ctx, p, C.byref(ptr)), st.ctx)
                    S = nx.shard_len(table[p].numel, world)
                    got = rt.view(ptr.value, world * S, torch.bfloat16).view(torch.int16).cpu().numpy()
                    ref = nx.all_gather_padded([nx.bf16_bits(nx.shard_of(full[p], world, q)) for q in range(world)])
                    assert np.array_equal(got.view(np.uint16), ref), (st.rank, p)
                    checked.append(p)
        elif o["kind"] == "rel":
            for st in ranks.values():
                dc.check(dc.lib.dc_release(st.ctx, o["id"], st.streams[0].cuda_stream), st.ctx)
    torch.cuda.synchronize()
    rt.poll(ranks)
    assert sorted(set(checked)) == list(range(len(table)))


@pytest.mark.parametrize("world,passes", [(2, dc.DC_PASS_SHARD), (4, dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH),
                                          (8, dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD)])
def test_ag_push_virtual_ranks(world, passes):
    cfg = synth.small_llama(layers=2, seq=128)
    table = synth.llama_param_table(cfg)
    ranks = rt.create_ranks(table, world)
    xs = {r: bf16_tensor(ost.rank_batch(cfg, r)[0]) for r in ranks}
    rt.attach_model(ranks, cfg, xs, xs)
    prof = rt.profile_json(ranks[0], tc=[[4096, 10], [1 << 20, 20], [1 << 26, 400]])
    M = 1 << 40
    sched = dc.plan(json.dumps(prof), M, M_prefetch=1 << 22, passes=passes, strict=True)
    rt.bind(ranks, {r: sched for r in ranks})
    full = ost.init_full_params(table)
    ops = _ops(sched)
    for st in ranks.values():
        dc.check(dc.lib.dc_step_begin(st.ctx, 1, st.streams[0].cuda_stream), st.ctx)
    checked = set()
    for o in ops:
        if o["kind"] == "ag":
            for st in ranks.values():
                ev = torch.cuda.Event()
                ev.record(st.streams[0])
                st.streams[1].wait_event(ev)
                dc.check(dc.lib.dc_gather(st.ctx, o["id"], st.streams[1].cuda_stream, None), st.ctx)
            torch.cuda.synchronize()
            for st in ranks.values():
                for p in o["members"]:
                    ptr = C.c_void_p()
                    dc.check(dc.lib.dc_tensor_ptr(st.ctx, p, C.byref(ptr)), st.ctx)
                    S = nx.shard_len(table[p].numel, world)
                    got = rt.view(ptr.value, world * S, torch.bfloat16).view(torch.int16).cpu().numpy()
                    ref = nx.all_gather_padded([nx.bf16_bits(nx.shard_of(full[p], world, q)) for q in range(world)])
                    assert np.array_equal(got.view(np.uint16), ref), (st.rank, p)
                    checked.add(p)
        elif o["kind"] == "rel":
            for st in ranks.values():
                dc.check(dc.lib.dc_release(st.ctx, o["id"], st.streams[0].cuda_stream), st.ctx)
    torch.cuda.synchronize()
    rt.poll(ranks)
    assert checked == set(range(len(table)))
    for st in ranks.values():
        assert dc.lib.dc_step_begin(st.ctx, 2, st.streams[0].cuda_stream) == dc.DC_OK   # no sticky timeout


# half-width tail units (pair kernel, forward-form GEMMs): when the tiles of the
# partial last wave fit twice over in one wave, each runs as two 256 x 128
# halves (UMMA N = 128).  sms = 8 -> 4 pairs; (M, N) = (512, 1280) -> 10 tiles =
# 2 waves of 4 + 2 tail tiles -> 4 half units.  Forward (K-major B, 2
# N-segments, residual, ragged N) against fp64; the dX / dW forms of the same
# shape (no half tails: MN-major operands) beside it.
@pytest.mark.parametrize("M,N,K", [(512, 1280, 512), (512, 1192, 320)])
def test_gemm_half_tail_units(M, N, K):
    sms = 8
    a, A = _mat(91, M, K)
    n1 = 512
    b1, B1 = _mat(92, n1, K)
    b2, B2 = _mat(93, N - n1, K)
    r, R = _mat(94, M, N)
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, K, A, K, 0, [B1, B2], [K, K], [n1 // 256, -(-N // 256)], 0, 0, Cm, N, R=R, ldr=N, sms=sms, kernel=2)
    bcat = np.concatenate([b1, b2])
    _check(Cm, a @ bcat.T + r, np.abs(a) @ np.abs(bcat).T + np.abs(r), "half-tail fwd")
    k1 = (K // 2) // 64 * 64
    w1, W1 = _mat(95, k1, N)
    w2, W2 = _mat(96, K - k1, N)
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, K, A, K, 0, [W1, W2], [N, N], [k1 // 64, -(-K // 64)], 1, 1, Cm, N, sms=sms, kernel=2)
    wcat = np.concatenate([w1, w2])
    _check(Cm, a @ wcat, np.abs(a) @ np.abs(wcat), "half-tail dx")
    dy, DY = _mat(97, K, M)
    x, X = _mat(98, K, N)
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(M, N, K, DY, M, 1, [X], [N], [0], 1, 0, Cm, N, sms=sms, kernel=2)
    _check(Cm, dy.T @ x, np.abs(dy).T @ np.abs(x), "half-tail dw")
