"""N > 1 host logic on CPU (world size 2, gloo): each rank profiles
differently, the profile is MAX-reduced (reading D12), every rank runs dc_plan
(host-only C++) and the resulting canonical schedules must be byte-identical
across ranks and equal to the oracle's plan of the reduced profile."""
import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import numerics as nx
from oracle import sched as osd
from tests import sched_util as su


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _profile(rank):
    cfg = synth.small_llama(layers=3)
    comp = synth.models.llama_compute_ops(cfg)
    s0 = osd.build_s0(comp)
    world = 2
    B = {p.id: nx.shard_len(p.numel, world) * world * 2 for p in synth.llama_param_table(cfg)}
    live = osd.live_before_s0(s0, B)
    act, pm = 0, {}
    for o in s0:
        pm[o["id"]] = 10 ** 6 + act + live[o["id"]] + 4096 * rank * (o["id"] % 7)   # rank-dependent noise
        if o["kind"] == "compute":
            act += 50000 if o["phase"] == "fwd" else -50000
            act = max(act, 0)
    return su.make_profile([(o["name"], o["kind"], o["phase"], o["micro"], o["layer"], o["params"]) for o in comp],
                           B, pm, dur=lambda o: 10 + o["id"] % 5, tc=[[4096, 20 + rank], [1 << 20, 40], [1 << 24, 300]])


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_09983_b200 import dc, runtime as rt
    prof = rt.max_reduce_profile(_profile(rank), dist.group.WORLD)
    M = max(o["p_mem"] for o in prof["ops"]) + 3 * 10 ** 6
    sched = dc.plan(json.dumps(prof), M, M_prefetch=1 << 20, strict=True)
    js = dc.schedule_json(sched)
    digests = [None] * world
    dist.all_gather_object(digests, rt.plan_digest(js))
    with open(os.path.join(out_dir, "r%d.json" % rank), "w") as f:
        json.dump({"digests": digests, "plan": js, "profile": prof, "M": M}, f)
    dist.destroy_process_group()


def test_two_ranks_plan_identically(tmp_path):
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, start_method="spawn")
    r0 = json.load(open(tmp_path / "r0.json"))
    r1 = json.load(open(tmp_path / "r1.json"))
    assert r0["digests"][0] == r0["digests"][1] == r1["digests"][0]
    assert r0["plan"] == r1["plan"]
    # the reduced profile really is the element-wise max of the two local ones
    p0, p1 = _profile(0), _profile(1)
    for a, b, c in zip(p0["ops"], p1["ops"], r0["profile"]["ops"]):
        assert c["p_mem"] == max(a["p_mem"], b["p_mem"])
    assert r0["profile"]["tc"][0][1] == 21
    # and equals the oracle's plan of that profile, byte for byte
    oracle = osd.canonical_json(osd.plan(r0["profile"], r0["M"], 1 << 20, strict=True))
    assert oracle == r0["plan"]
