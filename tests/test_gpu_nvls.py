"""NVLS collectives: the multimem.st all-gather and the
multimem.ld_reduce reduce-scatter + Adam (csrc/nvls.cu, option "nvls",
dc_bind_multicast).

* Gating, on any box: virtual ranks have no multicast mapping, so
  dc_bind_multicast refuses non-zero addresses there, and with option "nvls"
  set but no multicast address bound the library runs the unicast kernels —
  two planned N = 2 steps checked against the oracle.
* The NVLS kernels themselves need >= 2 GPUs on an NVSwitch whose driver
  grants multicast objects (torch symmetric memory's multicast_ptr != 0):
  two processes, one per GPU, run planned steps with multimem gathers (update
  bit-exact against the oracle's reduce-scatter + Adam of the GPUs' own grads)
  and then with the switch-side reduce-scatter (not bit-exact: the switch sums
  in its own order and returns bf16; the master update is checked within the
  north star's bf16 tolerance of the update it stands for).  Skipped, with
  the reason, on boxes without that.
"""
import json
import os
import socket

import numpy as np
import pytest
import torch

import synth
from oracle import step as ost
from tests.gpu_util import bf16_tensor
from tests.oracle_check import check_step

pytestmark = pytest.mark.gpu

dc = pytest.importorskip("paper_2504_09983_b200.dc")
from paper_2504_09983_b200 import runtime as rt  # noqa: E402

LR = 1e-3
TC = [[4096, 10], [1 << 20, 20], [1 << 26, 400]]


def test_nvls_gated_off_without_multicast():
    cfg = synth.small_llama(layers=2, seq=128)
    table = synth.llama_param_table(cfg)
    ranks = rt.create_ranks(table, 2, lr=LR)
    xs, ts = {}, {}
    for r in ranks:
        x, t = ost.rank_batch(cfg, r)
        xs[r], ts[r] = bf16_tensor(x), bf16_tensor(t)
    rt.attach_model(ranks, cfg, xs, ts)
    st0 = ranks[0]
    assert dc.lib.dc_bind_multicast(st0.ctx, 0, 0, 0) == dc.DC_ESTATE          # no schedule yet
    assert dc.lib.dc_set_option(st0.ctx, b"nvls", 4) == dc.DC_EINVAL
    prof = rt.profile_json(st0, tc=TC)
    sched = dc.plan(json.dumps(prof), 1 << 40, M_prefetch=1 << 22,
                    passes=dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD, strict=True)
    rt.bind(ranks, {r: sched for r in ranks})
    for st in ranks.values():
        assert dc.lib.dc_bind_multicast(st.ctx, 1 << 20, 0, 1 << 21) == dc.DC_EINVAL   # virtual ranks
        assert dc.lib.dc_bind_multicast(st.ctx, 1 << 20, 0, 0) == dc.DC_EINVAL         # no flag address
        dc.check(dc.lib.dc_bind_multicast(st.ctx, 0, 0, 0), st.ctx)
        dc.check(dc.lib.dc_set_option(st.ctx, b"nvls", 3), st.ctx)
    for s in (1, 2):   # unicast kernels run: exact against the oracle
        check_step(ranks, table, cfg, 2, s, LR, lambda: rt.step(ranks, s))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    from oracle import numerics as nx
    from tests.gpu_util import slot_grads
    from tests.oracle_check import snapshot
    res = {"multicast": False}
    try:
        cfg = synth.small_llama(layers=2, seq=128)
        table = synth.llama_param_table(cfg)
        ranks = rt.create_ranks(table, world, rank, virtual=False, group=dist.group.WORLD, rank=rank, lr=LR)
        st = ranks[rank]
        res["multicast"] = bool(rt.multicast_ptr(st.peer_keep["flags"]))
        x, t = ost.rank_batch(cfg, rank)
        rt.attach_model(ranks, cfg, {rank: bf16_tensor(x, dev)}, {rank: bf16_tensor(t, dev)})
        prof = rt.max_reduce_profile(rt.profile_json(st, tc=TC), dist.group.WORLD, device=dev)
        sched = dc.plan(json.dumps(prof), 1 << 40, M_prefetch=1 << 22,
                        passes=dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH | dc.DC_PASS_UNSHARD, strict=True)
        rt.bind(ranks, {rank: sched}, group=dist.group.WORLD)
        if res["multicast"]:
            res["bits"] = []
            for step, bits in ((1, 1), (2, 3)):
                info = rt.bind_multicast(st, bits)
                res["bits"].append(info)
                before = snapshot(ranks, table)
                rt.step(ranks, step)
                torch.cuda.synchronize()
                rt.poll(ranks)
                after = snapshot(ranks, table)
                g = slot_grads(st, table, world, layers={0, 1})
                allg = [None] * world                     # every rank's grads (host) for the oracle RS
                dist.all_gather_object(allg, g)
                worst = 0.0
                for i, p in enumerate(table):
                    b, a = before[rank][i], after[rank][i]
                    e_mst = nx.rs_adam_shard([allg[q][i] for q in range(world)], b["master"], b["m"], b["v"],
                                             world, rank, step, LR)[0]
                    if bits & 2:          # switch-side sum: within 2e-2 of the update it stands for
                        upd = np.abs(np.asarray(e_mst, np.float64) - b["master"])
                        tol = 2e-2 * upd + 2 * np.spacing(np.abs(np.asarray(e_mst, np.float32))).astype(np.float64)
                        d = np.abs(a["master"].astype(np.float64) - e_mst)
                        worst = max(worst, float((d / np.maximum(tol, 1e-30)).max()))
                    else:                 # multimem gathers: the step is the unicast step, bit for bit
                        assert a["master"].tobytes() == np.asarray(e_mst, np.float32).tobytes(), (step, p.name)
                res.setdefault("worst", []).append(worst)
        res["ok"] = True
    except Exception as e:   # reported to the parent
        res["error"] = repr(e)
    with open(os.path.join(out_dir, "r%d.json" % rank), "w") as f:
        json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2,
                    reason="NVLS needs >= 2 GPUs on one NVSwitch (this box has %d); the one-GPU driver refuses "
                           "cuMulticastCreate (profiles/r01g/nvls/probe.txt)" % torch.cuda.device_count())
def test_nvls_two_gpus(tmp_path):
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    r = [json.load(open(tmp_path / ("r%d.json" % q))) for q in range(2)]
    for q in range(2):
        assert r[q].get("ok"), r[q]
    if not r[0]["multicast"]:
        pytest.skip("torch symmetric memory gave no multicast address on this box (no NVLS)")
    for q in range(2):
        assert r[q]["bits"][0]["ag_multimem"] and r[q]["bits"][1]["rs_ld_reduce"], r[q]
        assert max(r[q]["worst"]) <= 1.0, r[q]
