"""Error behaviour of the C ABI on the GPU (include/dc.h conventions): state
errors before binding, argument errors, and a peer that never arrives — the
bounded device flag wait times out, sets the sticky error word, the kernels
finish (no hang) and the next call reports DC_ETIMEOUT."""
import ctypes as C
import json
import time

import pytest
import torch

import synth
from oracle import step as ost
from tests.gpu_util import bf16_tensor

pytestmark = pytest.mark.gpu

dc = pytest.importorskip("paper_2504_09983_b200.dc")
from paper_2504_09983_b200 import runtime as rt  # noqa: E402


def test_state_and_argument_errors():
    cfg = synth.small_llama(layers=2, seq=128)
    table = synth.param_table(cfg)
    st = rt.create_ranks(table, 2)[0]
    cs = st.streams[0].cuda_stream
    assert dc.lib.dc_gather(st.ctx, 0, cs, None) == dc.DC_ESTATE            # no schedule bound
    assert dc.lib.dc_reduce_scatter_step(st.ctx, 5, 1, 0, cs) == dc.DC_EINVAL   # bad layer
    assert dc.lib.dc_reduce_scatter_step(st.ctx, 0, 0, 0, cs) == dc.DC_EINVAL   # step_t is 1-based
    assert dc.lib.dc_reduce_scatter_step(st.ctx, 0, 1, 0, cs) == dc.DC_ESTATE   # slot never acquired
    d = dc.ModelDims(cfg.hidden, cfg.ffn, cfg.n_heads, cfg.n_kv, cfg.head_dim, cfg.layers, cfg.tokens, 0, 0)
    m = C.c_void_p()
    dc.check(dc.lib.dc_model_create(st.ctx, C.byref(d), C.byref(m)))
    need = C.c_uint64()
    dc.check(dc.lib.dc_model_act_bytes(m, C.byref(need)))
    buf = torch.empty(need.value, dtype=torch.uint8, device="cuda")
    x = torch.zeros(cfg.tokens * cfg.hidden, dtype=torch.bfloat16, device="cuda")
    assert dc.lib.dc_model_step(m, 1, 0, cs, cs, cs, cs) == dc.DC_ESTATE      # not bound
    assert dc.lib.dc_model_bind(m, buf.data_ptr(), need.value - 256, x.data_ptr(), x.data_ptr()) == dc.DC_EOOM
    assert dc.lib.dc_model_bind(m, buf.data_ptr() + 8, need.value, x.data_ptr(), x.data_ptr()) == dc.DC_EINVAL
    dc.check(dc.lib.dc_model_bind(m, buf.data_ptr(), need.value, x.data_ptr(), x.data_ptr()))
    assert dc.lib.dc_model_step(m, 1, 0, cs, cs, cs, cs) == dc.DC_ESTATE      # no schedule bound
    assert dc.lib.dc_model_set_option(m, b"fuse_act", 7) == dc.DC_EINVAL
    dc.lib.dc_model_destroy(m)


def test_missing_peer_times_out_without_hanging():
    """Rank 1 of 2 never steps: rank 0's first gather waits for rank 1's ready
    flag, gives up after spin_limit (0.3 s), and the failure surfaces as
    DC_ETIMEOUT from dc_poll / the next call; the GPU stays usable."""
    cfg = synth.small_llama(layers=2, seq=128)
    table = synth.param_table(cfg)
    ranks = rt.create_ranks(table, 2, spin_ms=300)
    xs, ts = {}, {}
    for r in ranks:
        x, t = ost.rank_batch(cfg, r)
        xs[r], ts[r] = bf16_tensor(x), bf16_tensor(t)
    rt.attach_model(ranks, cfg, xs, ts)
    prof = rt.profile_json(ranks[0])
    sched = dc.plan(json.dumps(prof), 1 << 40, passes=dc.DC_PASS_SHARD)
    rt.bind(ranks, {r: sched for r in ranks})
    st = ranks[0]
    t0 = time.time()
    dc.check(dc.lib.dc_model_step(st.model, 1, 0, *st.stream_handles()), st.ctx)   # enqueue only
    torch.cuda.synchronize()                       # completes: every wait is bounded
    assert time.time() - t0 < 60
    assert dc.lib.dc_poll(st.ctx) == dc.DC_ETIMEOUT
    assert "timed out" in dc.last_error(st.ctx)
    assert dc.lib.dc_model_step(st.model, 2, 0, *st.stream_handles()) == dc.DC_ETIMEOUT   # sticky
    a = torch.ones(1024, device="cuda")
    assert float((a * 2).sum()) == 2048.0          # the device still runs work
