"""The one-process-per-GPU path (virtual=False) on torch symmetric memory:
grad slots and flag table come from torch.distributed._symmetric_memory
(empty + rendezvous over an NCCL group), which is what bench.py uses at N > 1
on an NVSwitch box.  On a one-GPU box the group has one rank; the step through
the C ABI is checked against the oracle (tests/oracle_check.py)."""
import json
import os

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


def test_symmetric_memory_rank_step():
    import torch.distributed as dist
    assert rt.symm_backend() == "symm_mem"
    store = dist.HashStore()
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        group = dist.group.WORLD
        cfg = synth.small_llama(layers=2, seq=128)
        table = synth.llama_param_table(cfg)
        ranks = rt.create_ranks(table, 1, 0, virtual=False, group=group, rank=0, lr=LR)
        st = ranks[0]
        assert set(st.peer_keep) == {"grad", "flags"}
        # the symmetric buffers map to this rank's own tensors
        g, f = st.tensors["grad"], st.tensors["flags"]
        assert int(st.peer_keep["grad"][0].buffer_ptrs[0]) == g.data_ptr()
        assert int(st.peer_keep["flags"][0].buffer_ptrs[0]) == f.data_ptr()
        x, t = ost.rank_batch(cfg, 0)
        rt.attach_model(ranks, cfg, {0: bf16_tensor(x)}, {0: bf16_tensor(t)})
        prof = rt.profile_json(st)
        sched = dc.plan(json.dumps(prof), 1 << 40, passes=dc.DC_PASS_SHARD | dc.DC_PASS_PREFETCH, strict=True)
        rt.bind(ranks, {0: sched}, group=group)
        for step in (1, 2):
            check_step(ranks, table, cfg, 1, step, LR, lambda: rt.step(ranks, step))
    finally:
        dist.destroy_process_group()


def test_symm_backend_has_no_silent_fallback(monkeypatch):
    monkeypatch.setenv("DC_SYMM", "nvshmem")
    with pytest.raises(ValueError):
        rt.symm_backend()
    monkeypatch.setenv("DC_SYMM", "ipc")
    assert rt.symm_backend() == "ipc"
    assert os.environ["DC_SYMM"] == "ipc"


def test_symm_mem_refusal_is_reported_not_silent(monkeypatch):
    """Without an explicit DC_SYMM, a runtime that refuses torch symmetric
    memory gets CUDA IPC peer mappings AND the reason in symm_backend() (bench
    puts it in collectives.transport); with DC_SYMM=symm_mem it raises."""
    import torch.distributed as dist
    from torch.distributed import _symmetric_memory as symm_mem

    def refuse(*a, **k):
        raise RuntimeError("symmetric memory refused (test)")

    monkeypatch.setattr(symm_mem, "empty", refuse)
    monkeypatch.delenv("DC_SYMM", raising=False)
    store = dist.HashStore()
    dist.init_process_group("gloo", store=store, rank=0, world_size=1)
    try:
        dev = torch.device("cuda", 0)
        monkeypatch.setenv("DC_SYMM", "symm_mem")
        with pytest.raises(RuntimeError):
            rt._alloc_symmetric(4096, dist.group.WORLD, dev)
        monkeypatch.delenv("DC_SYMM")
        t, ptrs, keep = rt._alloc_symmetric(4096, dist.group.WORLD, dev)
        assert ptrs == [t.data_ptr()] and t.numel() == 4096
        assert rt.symm_backend().startswith("ipc (torch symmetric memory unavailable: RuntimeError")
    finally:
        rt.SYMM_FALLBACK = None
        dist.destroy_process_group()
