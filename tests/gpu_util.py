"""Shared helpers for the -m gpu parity tests (no method arithmetic)."""
import numpy as np
import torch

import synth
from oracle import numerics as nx


def bf16_tensor(a_f32, device="cuda"):
    """fp32 numpy -> bf16 torch on device, RNE (same rounding as the oracle)."""
    bits = nx.bf16_bits(np.asarray(a_f32, np.float32))
    return torch.from_numpy(bits.view(np.int16).copy()).to(device).view(torch.bfloat16)


def to_np(t):
    """torch (any float dtype, any device) -> float64 numpy."""
    return t.detach().float().cpu().numpy().astype(np.float64)


def seeded(seed, tid, n, std=1.0):
    return synth.values(seed, tid, 0, n, synth.std_to_k(std))


def rel_norm(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


# ---------------------------------------------------------------- element-wise checks
def ulp_bf16(x):
    """Spacing of bf16 numbers at |x| (2^(e-7) for |x| in [2^e, 2^(e+1)))."""
    x = np.maximum(np.abs(np.asarray(x, np.float64)), 2.0 ** -126)
    return 2.0 ** (np.floor(np.log2(x)) - 7)


def assert_bf16_close(got, ref, name, rel=2e-2, ulps=4, rows=None):
    """Element-wise: |got - ref| <= rel |ref| + ulps * ulp_bf16(max |ref| of the
    element's row).  `rows`: reshape both to (rows, -1) first (default: one
    row).  The absolute term admits the rounding of a bf16 result whose value
    cancelled below its row's scale (a GEMM output is a sum of products of the
    row's magnitude); a wrong element, row or sign fails it."""
    g = np.asarray(got, np.float64)
    r = np.asarray(ref, np.float64)
    assert g.shape == r.shape or g.size == r.size, (name, g.shape, r.shape)
    g = g.reshape(rows if rows else 1, -1)
    r = r.reshape(g.shape)
    scale = ulp_bf16(np.abs(r).max(axis=1, keepdims=True))
    tol = rel * np.abs(r) + ulps * scale
    err = np.abs(g - r)
    bad = ~(err <= tol)                     # NaN fails
    if bad.any():
        i = np.unravel_index(np.argmax(np.where(bad, err / np.maximum(tol, 1e-300), -1)), g.shape)
        raise AssertionError("%s: %d of %d elements outside tolerance; worst at %s: got %r ref %r (tol %g)" %
                             (name, int(bad.sum()), g.size, tuple(int(k) for k in i), g[i], r[i], tol[i]))
    return float((err / np.maximum(tol, 1e-300)).max()) if err.size else 0.0


def slot_grads(st, table, world, layers=None):
    """bf16 padded full gradients left in this rank's grad slots after a step
    (layer l in slot l % 2; valid for the last two layers of the backward)."""
    import ctypes as C

    from paper_2504_09983_b200 import dc, runtime as rt
    out = {}
    for i, p in enumerate(table):
        if layers is not None and p.layer not in layers:
            continue
        slot = C.c_void_p()
        dc.check(dc.lib.dc_grad_slot(st.ctx, p.layer, C.byref(slot)), st.ctx)
        S = nx.shard_len(p.numel, world)
        t = rt.view(slot.value + rt.grad_offset(st, i), world * S, torch.bfloat16)
        out[i] = t.float().cpu().numpy()
    return out


def assert_update_exact(ranks, table, before, grads, step, lr, params=None):
    """The fp32 master / m / v and the bf16 shard after a step equal, bit for
    bit, the oracle's reduce-scatter + 1/N + Adam (oracle.numerics.rs_adam_shard)
    applied to the states before the step and the ranks' own bf16 grads
    (`grads[q][i]`, padded full tensors) — the update is checked exactly, the
    grads themselves separately against the oracle's."""
    from paper_2504_09983_b200 import runtime as rt
    world = len(grads)
    for r, st in ranks.items():
        got = {k: st.tensors[k].cpu().numpy() for k in ("master", "m", "v")}
        sh = st.tensors["shard"].view(torch.int16).cpu().numpy().view(np.uint16)
        for i, p in enumerate(table):
            if params is not None and i not in params:
                continue
            off, n = rt.shard_range(st, i)
            mst, m, v = (before[k][r][i] for k in ("master", "m", "v"))
            e_mst, e_m, e_v, e_sh = nx.rs_adam_shard([grads[q][i] for q in range(world)], mst, m, v, world, r,
                                                     step, lr)
            for k, e in (("master", e_mst), ("m", e_m), ("v", e_v)):
                assert got[k][off:off + n].tobytes() == np.asarray(e, np.float32).tobytes(), (r, p.name, k)
            assert np.array_equal(sh[off:off + n], nx.bf16_bits(e_sh)), (r, p.name, "shard")


def states_of(ranks, table):
    """{master|m|v: [rank][param] fp32 numpy shard} snapshot of the device states."""
    from paper_2504_09983_b200 import runtime as rt
    out = {k: {} for k in ("master", "m", "v")}
    for r, st in ranks.items():
        for k in out:
            a = st.tensors[k].cpu().numpy()
            out[k][r] = []
            for i in range(len(table)):
                off, n = rt.shard_range(st, i)
                out[k][r].append(a[off:off + n].copy())
    return out
