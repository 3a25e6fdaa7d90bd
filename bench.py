"""Benchmark: the sharded training step of a Llama-3-8B-shaped layer stack
(BASELINE.json configs[1]) through the C ABI, one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--layers L]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the CPU oracle, same metric/config

With --gpus N > 1 and no RANK in the environment, bench.py launches itself
once per GPU through torch.distributed.run (127.0.0.1, a free port) and passes
rank 0's JSON line through; under torchrun it runs as one rank.

Flow (§3 / §5.5): S_0 warm-up steps (5) with per-op profiling
-> profile MAX-reduced over ranks -> dc_plan (prefetch + unshard, strict) ->
W warm-up steps -> K timed steps (CUDA events on the compute stream, barrier +
synchronize on both sides, max over ranks) -> K end-to-end steps with pinned
host inputs copied in and the loss read back -> CPU oracle sample.
Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/sec/box (device-timed, max over ranks) at 1/2/4/8 B200; AG/RS GB/s vs 900 GB/s"
GiB = 1 << 30
# model -> (synth config name, default layers on one GPU, BASELINE config it stands for)
MODELS = {
    "llama3-8b": ("LLAMA3_8B", 32, "BASELINE configs[1]"),
    # 14 B of state per parameter: 70B L=8 (96 GB) and Mixtral L=4 (81 GB) fit
    # one 180 GB B200; the full stacks are the 8-GPU configs[2] / configs[3]
    "llama3-70b": ("LLAMA3_70B", 8, "BASELINE configs[2] layer shapes"),
    "mixtral-8x7b": ("MIXTRAL_8X7B", 4, "BASELINE configs[3] layer shapes"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=2)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--model", default="llama3-8b", choices=sorted(MODELS),
                    help="layer shapes (PAPER.md line 440 / BASELINE configs)")
    ap.add_argument("--layers", type=int, default=0, help="0: the model's default for one GPU")
    ap.add_argument("--micro", type=int, default=1, help="gradient-accumulation micro-steps per step (P:362)")
    ap.add_argument("--checkpoint", action="store_true", help="layer-level activation checkpointing (P:440)")
    ap.add_argument("--passes", default="PS", help="S0 | P | S | PS")
    ap.add_argument("--offload", action="store_true",
                    help="adaptive offload of optimizer states (Alg. 2, P:370-408) with host-resident fragments "
                         "(reading D28): BASELINE configs[4], e.g. --model llama3-70b --layers 16 --batch 1")
    ap.add_argument("--offload-sync", action="store_true",
                    help="the paper's comparison point for --offload (P:504-506): every optimizer-state fragment "
                         "host-resident, reloaded synchronously before its layer's update")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="capture one planned step as a CUDA graph (dc_model_graph_capture) and replay it in the "
                         "timed and e2e loops (dc_model_graph_launch); auto = at N = 1 (measured there), on = at "
                         "any N (per-step device barrier + flag reset)")
    ap.add_argument("--no-graph", action="store_true", help="same as --graph off")
    ap.add_argument("--share-gpu", action="store_true",
                    help="test mode: every rank on cuda:0 (gloo host collectives, CUDA-IPC peer maps, fixed T_c); "
                         "exercises the N > 1 launch on a one-GPU box, numbers are not a bench value")
    ap.add_argument("--profile-json", default="", help="write the rank-0 profile / plan here")
    ap.add_argument("--tc-table", default="",
                    help="plan with this T_c(V) table instead of the measured / zero one (what-if, SURVEY §8 a-3): "
                         "a JSON file [[bytes, us], ...], or SWEEP.json:N:mode to take the median times of "
                         "scripts/ag_sweep.py's run at N virtual ranks (mode sm | ce)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without a GPU: every rank joins a gloo group, barriers, MAX-reduces a "
                         "dummy time and rank 0 prints one JSON line (tests/test_bench_cli.py)")
    return ap.parse_args()


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args):
    """--gpus N > 1 outside torchrun: one process per GPU through
    torch.distributed.run on this node (rendezvous on 127.0.0.1).  stdout of
    the ranks is passed through (only rank 0 prints the JSON line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % args.gpus,
           "--master-addr=127.0.0.1", "--master-port=%d" % free_port(), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(cmd, env=env)


def dry_run(args):
    """The N-rank plumbing of the GPU arm with no GPU work: rank / world from
    the launcher, gloo group, barrier, MAX over ranks, one JSON line."""
    import torch
    import torch.distributed as dist
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit("bench: WORLD_SIZE %d != --gpus %d" % (world, args.gpus))
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    seen = [(rank, os.getpid())]
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        seen = [None] * world
        dist.all_gather_object(seen, (rank, os.getpid()))
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "max_over_ranks": t.item(),
                          "ranks": [r for r, _ in seen], "processes": len({p for _, p in seen})}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def peaks():
    p = {"hbm_gbs": 6546.6, "bf16_tflops": 1647.5, "bf16_tflops_sustained": 1402.6, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured (MEASURED_PEAKS.json)"
    except (OSError, ValueError):
        pass
    return p


# ----------------------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(", ") for r in out.strip().splitlines() if r.count(",") >= 7]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].strip() == "Active"})
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        pw = []
        for r in rows:
            try:
                pw.append(float(r[3]))
            except ValueError:
                pass
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w": {"median": statistics.median(pw), "max": max(pw)} if pw else None}


BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


# ----------------------------------------------------------------------------- oracle sample
class OracleSample:
    """The CPU oracle on a bounded sample of the workload: ONE layer of the
    stack, N=1, at T tokens (T <= max_tokens) — forward + backward
    (bf16-emulated, fp64 GEMMs) + reduce-scatter + Adam over the layer's
    218 M parameters.  Weights are generated once (untimed); step(T) returns
    seconds.

    Extrapolation to the workload (documented in DESIGN.md §9): one layer
    sample costs t(T) = a + b T — the reduce-scatter + Adam pass over the
    layer's parameters does not depend on T (a), the layer's forward and
    backward GEMMs / glue are linear in T (b).  a and b come from the medians
    of samples at two token counts; the L-layer step at the workload's T_w
    tokens then takes L (a + b T_w)."""

    def __init__(self, cfg, max_tokens):
        import synth
        from oracle import numerics as nx
        self.cfg, self.t = cfg, 0
        self.table = synth.llama_param_table(cfg)[:9]
        self.W, self.masters = {}, []
        for p in self.table:
            v = (np.ones(p.numel, np.float32) if p.k == 0.0 else synth.values(0, p.id, 0, p.numel, p.k))
            self.masters.append(v)
            self.W[p.name] = nx.rne_bf16(v).reshape(p.shape)
        n = max_tokens * cfg.hidden
        self.x = nx.rne_bf16(synth.values(1000, 0, 0, n, synth.K_UNIT)).reshape(max_tokens, cfg.hidden)
        self.y_t = nx.rne_bf16(synth.values(2000, 0, 0, n, synth.K_UNIT)).reshape(max_tokens, cfg.hidden)
        self.ms = [np.zeros_like(v) for v in self.masters]
        self.vs = [np.zeros_like(v) for v in self.masters]
        self.secs = {}

    def step(self, tokens):
        from oracle import model as om
        from oracle import numerics as nx
        self.t += 1
        t0 = time.perf_counter()
        y, c = om.llama_layer_fwd(self.x[:tokens], self.W, self.cfg, nx.rne_bf16)
        _, dy = om.mse_loss(y, self.y_t[:tokens])
        _, G = om.llama_layer_bwd(nx.rne_bf16(dy), c, self.W, self.cfg, nx.rne_bf16)
        for i, p in enumerate(self.table):
            g = nx.reduce_scatter([np.asarray(G[p.name], np.float32).reshape(-1)], 1, 0)
            self.masters[i], self.ms[i], self.vs[i] = nx.adam_update(
                self.masters[i], self.ms[i], self.vs[i], nx.scale_mean(g, 1), self.t)
        sec = time.perf_counter() - t0
        self.secs.setdefault(tokens, []).append(sec)
        return sec

    def fit(self):
        """(a, b) of t(T) = a + b T from the per-T medians (two token counts)."""
        (t1, s1), (t2, s2) = sorted((t, statistics.median(v)) for t, v in self.secs.items())[:2]
        b = max((s2 - s1) / (t2 - t1), 1e-12)
        a = max(s1 - b * t1, 0.0)
        return a, b

    def tokens_per_s(self, cfg):
        """Extrapolated tokens/s of the L-layer step at the workload's tokens."""
        a, b = self.fit()
        return cfg.tokens / (cfg.layers * (a + b * cfg.tokens)), a, b


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) on host cores.
    A step is one layer sample, alternating 32 and 64 tokens (warm-up covers
    both); `ms_per_step` is the measured time of those samples, `value` the
    tokens/s of the workload extrapolated with OracleSample's model."""
    import synth  # noqa: F401
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.model != "llama3-8b":
        print(json.dumps({"impl": "reference", "unavailable": "the oracle sample is defined for the default "
                          "llama3-8b workload only (a 70B / Mixtral layer's states exceed a bounded CPU sample)"}))
        return
    cfg = model_config(args)
    sizes = (32, 64)
    sample_run = OracleSample(cfg, max(sizes))
    for i in range(max(args.warmup, 2)):
        sample_run.step(sizes[i % 2])
    sample_run.secs = {} if args.steps >= 2 else sample_run.secs
    secs = [sample_run.step(sizes[i % 2]) for i in range(args.steps)]
    per_step = float(np.mean(secs))
    val, a, b = sample_run.tokens_per_s(cfg)
    sample = ("1 Llama-3-8B-shaped layer at %d / %d tokens alternating, N=1: oracle fwd+bwd+RS+Adam; measured "
              "t(T) = a + b T per layer with a = %.2f s (RS + Adam, token-independent), b = %.4f s/token; "
              "workload %d layers x %d tokens -> %.0f s per step" %
              (sizes[0], sizes[1], a, b, cfg.layers, cfg.tokens, cfg.layers * (a + b * cfg.tokens)))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
            "ms_per_step_note": "measured wall time of one step = one layer sample (not the extrapolated "
                                "workload step; see cpu_baseline.sample)",
            "extrapolated_ms_per_workload_step": cfg.layers * (a + b * cfg.tokens) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (oracle)",
            "data": "synthetic",
            "config": {"workload": "llama3-8b-stack (BASELINE configs[1]), oracle sample", "seq_len": args.seq,
                       "global_batch": args.batch, "layers": cfg.layers},
            "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def _base_op(name):
    """exp_gu_3 -> exp_gu (per-expert MoE ops carry the expert index)."""
    head, _, tail = name.rpartition("_")
    return head if tail.isdigit() else name


def gemm_flops(name, cfg, T):
    """2 M N K of the op's GEMMs (dX and dW in the backward); None for non-GEMM ops."""
    h, f, qd = cfg.hidden, cfg.ffn, cfg.q_dim
    qkvd = qd + 2 * cfg.kv_dim
    R = 2 * T // cfg.n_experts if cfg.n_experts else 0      # rows per expert (top-2, balanced)
    fwd = {"qkv": 2 * T * h * qkvd, "o_proj": 2 * T * qd * h, "gate_up": 2 * T * h * 2 * f, "down": 2 * T * f * h,
           "exp_gu": 2 * R * h * 2 * f, "exp_down": 2 * R * f * h}
    bwd = {k + "_bwd": 2 * v for k, v in fwd.items()}
    bwd["o_bwd"] = bwd.pop("o_proj_bwd")
    re = {"re_" + k: v for k, v in fwd.items()}          # checkpoint recompute
    return {**fwd, **bwd, **re}.get(_base_op(name))


def pcie_peaks(dev, torch, nbytes=1 << 30):
    """Pinned-host copy bandwidth (GB/s): H2D alone, D2H alone, and both at
    once on two streams (PCIe is full duplex) — the roofline of the offload
    path (BASELINE configs[4]).  Outside any timed region."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def run(h2d, d2h):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            if h2d:
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        return 3 * nbytes * (h2d + d2h) / (time.perf_counter() - t0) / 1e9

    run(True, True)
    out = {"h2d": run(True, False), "d2h": run(False, True), "duplex": run(True, True)}
    del h, h2, d, d2
    return {k: round(v, 1) for k, v in out.items()}


def tc_from_profile(prof):
    """T_c(V) of our own gather: in the profiled S_0 step every
    gather is one parameter, issued after its predecessor compute op finished
    (D23), and timed from "every receiver ready" to "every sender's stores
    landed".  Median per size, sizes ascending, made non-decreasing; integer us.
    None when the step timed no gathers (N = 1)."""
    B = {p["id"]: p["bytes"] for p in prof["params"]}
    by = {}
    for o in prof["ops"]:
        if o["kind"] == "ag" and o["dur_us"] > 0:
            by.setdefault(B[o["params"][0]], []).append(o["dur_us"])
    if not by:
        return None
    pts = [[b, int(statistics.median(v))] for b, v in sorted(by.items())]
    for i in range(1, len(pts)):
        pts[i][1] = max(pts[i][1], pts[i - 1][1])
    return pts


def measure_tc(group, world, dev, torch, dist):
    """T_c(V) table for the planner at N > 1: all-gather time vs full bytes,
    MAX over ranks (reading D12).  Measured with the NCCL comparator (same
    link), integer µs."""
    pts = []
    for lg in range(16, 31, 2):
        full = 1 << lg
        x = torch.empty(full // world // 2, dtype=torch.bfloat16, device=dev)
        out = torch.empty(full // 2, dtype=torch.bfloat16, device=dev)
        for _ in range(3):
            dist.all_gather_into_tensor(out, x, group=group)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            dist.all_gather_into_tensor(out, x, group=group)
        e1.record()
        torch.cuda.synchronize()
        us = torch.tensor([e0.elapsed_time(e1) * 1000 / 5], device=dev)
        dist.all_reduce(us, op=dist.ReduceOp.MAX, group=group)
        pts.append([full, max(1, int(round(us.item())))])
    for i in range(1, len(pts)):
        pts[i][1] = max(pts[i][1], pts[i - 1][1])
    del x, out
    torch.cuda.empty_cache()          # the sweep's buffers (up to 1 GiB) leave the allocator's cache
    return pts


def load_tc_table(spec):
    """--tc-table: [[bytes, us], ...] (integer us, strictly increasing bytes,
    made non-decreasing in time) from a file or from an ag_sweep.json run."""
    path, _, sel = spec.partition(":")
    with open(path) as f:
        d = json.load(f)
    if sel:
        n, _, mode = sel.partition(":")
        run = [r for r in d["runs"] if r["world"] == int(n) and r["mode"] == (mode or "sm")][0]
        pts = [[int(r["bytes"]), max(1, int(round(r["us"])))] for r in run["rows"]]
    else:
        pts = [[int(b), int(u)] for b, u in d]
    pts.sort()
    for i in range(1, len(pts)):
        pts[i][1] = max(pts[i][1], pts[i - 1][1])
    return pts


def model_config(args):
    import dataclasses

    import synth
    name, default_layers, _ = MODELS[args.model]
    return dataclasses.replace(getattr(synth, name), layers=args.layers or default_layers, seq=args.seq,
                               batch=args.batch)


def main():
    args = parse()
    if args.gpus > 1 and "RANK" not in os.environ and (args.impl == "ours" or args.dry_run):
        sys.exit(self_launch(args))
    if args.dry_run:
        dry_run(args)
        return
    if args.offload_sync:
        args.offload = True
    args.graph = not args.offload and not args.no_graph and args.graph != "off" and \
        (args.graph == "on" or args.gpus == 1)
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import synth
    from paper_2504_09983_b200 import dc, runtime as rt

    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if int(os.environ.get("WORLD_SIZE", "1")) != world:
        raise SystemExit("bench: WORLD_SIZE %s != --gpus %d" % (os.environ.get("WORLD_SIZE", "1"), world))
    if world > 1 and not args.share_gpu and torch.cuda.device_count() < world:
        raise SystemExit("bench: --gpus %d needs %d visible GPUs (found %d); --share-gpu runs the N-rank "
                         "flow on one GPU as a test" % (world, world, torch.cuda.device_count()))
    if world > 1:
        # communicator init lines (rank count, NVLS / P2P transport) on stderr,
        # which keeps stdout to the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.share_gpu:
        local = 0
        os.environ["DC_SYMM"] = "ipc"         # symmetric memory refuses two ranks on one device
        # processes time-slicing one GPU: keep one GEMM stream per process
        # (with the dW stream the pair's handshake intermittently stalled)
        os.environ.setdefault("DC_DW_CONCURRENT", "0")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # host-side collectives (barrier, MAX of timings / profiles) run on `cdev`
    cdev = torch.device("cpu") if args.share_gpu else dev
    group = None
    if world > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    cfg = model_config(args)
    T = cfg.tokens
    table = synth.param_table(cfg)
    lr = 1.5e-5
    n_micro = max(1, args.micro)
    if world == 1:
        ranks = rt.create_ranks(table, 1, local, virtual=True, lr=lr, micro_steps=n_micro,
                                defer_states=args.offload)
    else:
        ranks = rt.create_ranks(table, world, local, virtual=False, group=group, rank=rank, lr=lr,
                                micro_steps=n_micro, defer_states=args.offload)
    st = ranks[rank]
    if args.graph:
        dc.check(dc.lib.dc_set_option(st.ctx, b"graph_mode", 1), st.ctx)
    if os.environ.get("DC_AG_COPY_ENGINE") is not None:       # gathers on the copy engines (f-3)
        dc.check(dc.lib.dc_set_option(st.ctx, b"ag_copy_engine", int(os.environ["DC_AG_COPY_ENGINE"])), st.ctx)
    if os.environ.get("DC_FUSED_AG") is not None:             # fused all-gather -> GEMM (f-4)
        dc.check(dc.lib.dc_set_option(st.ctx, b"fused_ag", int(os.environ["DC_FUSED_AG"])), st.ctx)
    # synthetic inputs (synth generator, fp32) rounded to bf16 by torch (RNE)
    x_np = np.concatenate([synth.values(synth.seed_inputs(rank, mu), 0, 0, T * cfg.hidden, synth.K_UNIT)
                           for mu in range(n_micro)])
    t_np = np.concatenate([synth.values(synth.seed_targets(rank, mu), 0, 0, T * cfg.hidden, synth.K_UNIT)
                           for mu in range(n_micro)])
    x_host = torch.from_numpy(x_np).to(torch.bfloat16).pin_memory()
    t_host = torch.from_numpy(t_np).to(torch.bfloat16).pin_memory()
    x_dev = x_host.to(dev).view(n_micro, T, cfg.hidden)
    t_dev = t_host.to(dev).view(n_micro, T, cfg.hidden)
    rt.attach_model(ranks, cfg, {rank: x_dev}, {rank: t_dev}, checkpoint=args.checkpoint)
    for key in ("rs_overlap", "stream_k", "comm_sms"):          # A/B knobs (DC_RS_OVERLAP=0/1 ...)
        if os.environ.get("DC_" + key.upper()) is not None:
            dc.check(dc.lib.dc_model_set_option(st.model, key.encode(), int(os.environ["DC_" + key.upper()])))
    cs = st.streams[0]

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(group=group)

    # ---- S_0 warm-up + profile (five warm-up iterations, then profile)
    step_no = 0
    frags = None
    if args.offload:
        # the states do not fit beside the step, so S_0 cannot run: plan from
        # the executor's exact analytic P_mem (durations are not used by the
        # P / S / offload passes); whole (layer, m|v) fragments
        frags = rt.offload_fragments(st, rt.layer_state_bytes(table, world))
    else:
        # the fp32 m / v fragments define M_opt, which passes P and S add to the
        # profile's P_mem (reading D14); 256 MiB chunks (D15)
        frags = rt.offload_fragments(st, 256 << 20)
        prof0 = rt.profile_json(st)
        s0 = dc.plan(json.dumps(prof0), 1 << 50, passes=dc.DC_PASS_SHARD)
        rt.bind(ranks, {rank: s0}, group=group)
        for i in range(5):
            step_no += 1
            rt.step(ranks, step_no, profile=(i == 4))
    barrier()
    tc_nccl = None
    tc = tc_from_profile(rt.profile_json(st)) if world > 1 and not args.offload else None
    if world > 1 and not args.share_gpu:
        tc_nccl = measure_tc(group, world, dev, torch, dist)   # comparator (NCCL all-gather), reported
    if tc is None and world > 1:
        tc = tc_nccl or [[0, 20], [1 << 30, 20 + (1 << 30) // 100000]]
    elif tc is None:
        tc = [[0, 0], [1 << 40, 0]]
    if world > 1 and len(tc) < 2:
        tc = [[0, tc[0][1]], tc[0]]
    tc_source = ("our gathers in the profiled S_0 step" if world > 1 and tc is not tc_nccl else
                 "NCCL all-gather comparator" if world > 1 else "none (N = 1: gathers alias the shard)")
    if args.tc_table:
        tc, tc_source = load_tc_table(args.tc_table), "what-if: " + args.tc_table
    prof = rt.profile_json(st, tc=tc, frags=frags)
    if world > 1:   # element-wise MAX over ranks (reading D12)
        prof = rt.max_reduce_profile(prof, group, device=cdev)
    total = torch.cuda.get_device_properties(dev).total_memory
    M = int(0.9 * (total - 7 * GiB))
    passes = dc.DC_PASS_SHARD | (dc.DC_PASS_PREFETCH if "P" in args.passes else 0) | \
        (dc.DC_PASS_UNSHARD if "S" in args.passes and args.passes != "S0" else 0) | \
        (dc.DC_PASS_OFFLOAD | dc.DC_PASS_HOST_STATES if args.offload and not args.offload_sync else 0)
    t_plan = time.perf_counter()
    # offload-all-sync: no memory plan for the states (none stays on the device)
    sched = dc.plan(json.dumps(prof), (1 << 50) if args.offload_sync else M, passes=passes, strict=True)
    t_plan = time.perf_counter() - t_plan
    plan = json.loads(dc.schedule_json(sched))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(group=group)
    rt.bind(ranks, {rank: sched}, group=group)
    offload_info = None
    if args.offload:
        # extra ring slots (round-robin: a reload need not wait for the write-back
        # just issued) where the device has room beyond the plan, 6 GiB kept free
        fb = max(f["bytes"] for f in frags)
        if args.offload_sync:
            dc.check(dc.lib.dc_model_set_option(st.model, b"offload_all_sync", 1))
        off_bytes = sum(f["bytes"] for f in frags) if args.offload_sync else \
            sum(frags[i]["bytes"] for i in plan["offload"])
        free_b = torch.cuda.mem_get_info(dev)[0]
        dev_states = 2 * st.layout.shard_elems * 4 - off_bytes
        extra = int(max(0, min(2, (free_b - 6 * GiB - dev_states - 4 * fb) // fb)))
        mf, vf, pool, hb = rt.bind_host_states(ranks, alloc_host=True, extra_slots=extra)[rank]
        offload_info = {"mode": "all fragments, synchronous reload (P:504 baseline)" if args.offload_sync else
                        "adaptive (Alg. 2 + reload rule, host-resident fragments, D28)",
                        "pcie_peak_gbs": pcie_peaks(dev, torch),
                        "offloaded_bytes": off_bytes, "fragments": len(plan["offload"]),
                        "fragment_bytes": max(f["bytes"] for f in frags), "pool_bytes": pool,
                        "device_state_bytes": 4 * (2 * st.layout.shard_elems - mf - vf),
                        "pcie_bytes_per_step": 2 * off_bytes, "warnings": plan["warnings"][:4],
                        "n_warnings": len(plan["warnings"])}
    if world > 1:
        dist.barrier(group=group)
    if args.profile_json and rank == 0:
        with open(args.profile_json, "w") as f:
            json.dump({"profile": prof, "plan": plan, "M": M}, f)

    # ---- warm-up with the planned schedule
    for _ in range(max(3, args.warmup)):
        step_no += 1
        rt.step(ranks, step_no, profile=2 if args.graph else 0)   # graph: per-op events of an eager step
    barrier()
    if args.graph:
        try:
            dc.check(dc.lib.dc_model_graph_capture(st.model, step_no + 1, *st.stream_handles()), st.ctx)
        except dc.DCError as e:      # keep eager steps (same kernels, same results)
            print("bench: graph capture failed (%s); eager steps" % e, file=sys.stderr)
            args.graph = False
    if args.graph:
        for _ in range(2):                                       # replay warm-up
            step_no += 1
            dc.check(dc.lib.dc_model_graph_launch(st.model, step_no, cs.cuda_stream), st.ctx)
        barrier()

    def one_step(profile=0):
        if args.graph:
            dc.check(dc.lib.dc_model_graph_launch(st.model, step_no, cs.cuda_stream), st.ctx)
        else:
            rt.step(ranks, step_no, profile=profile)

    # ---- timed region (device-timed on the compute stream, max over ranks)
    def timed(k, profile_last=True):
        nonlocal step_no
        clocks = rt_clocks = None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        clk = Clocks(local)
        clk.start()
        time.sleep(0.3)
        e0.record(cs)
        launches = 0
        for i in range(k):
            step_no += 1
            one_step(profile=2 if (profile_last and i == k - 1) else 0)
            n = rt.C.c_int64()
            dc.check(dc.lib.dc_model_launch_count(st.model, rt.C.byref(n)))
            launches += n.value
        # host-resident states: the last step's state write-backs are inside the timed region
        dc.check(dc.lib.dc_model_join_states(st.model, cs.cuda_stream))
        e1.record(cs)
        barrier()
        clocks = clk.stop()
        rt.poll(ranks)
        ms = torch.tensor([e0.elapsed_time(e1) / k], device=cdev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
        return ms.item(), clocks, launches

    ms, clocks, launches = timed(args.steps)
    if clocks["reasons"] and BAD_REASONS & set(clocks["reasons"]):
        ms, clocks, launches = timed(args.steps)          # re-measure once
        clocks["remeasured"] = True
    last = rt.profile_json(st)        # per-op events of the last timed step (read before any other step)
    # host cost of enqueueing one step (diagnostic, outside the timed region):
    # if it approaches ms_per_step the step is launch-bound
    barrier()
    t_h = time.perf_counter()
    step_no += 1
    rt.step(ranks, step_no)
    host_enqueue_ms = (time.perf_counter() - t_h) * 1e3
    barrier()
    # one more step (outside the timed region) with the reduce-scatter + Adam in
    # compute-stream order: the GEMMs' own throughput without rs_adam holding
    # SMs (in the overlapped timed step a GEMM launched while rs_adam runs waits
    # for its CTAs, and that wait is inside the GEMM op's events)
    ov = int(os.environ.get("DC_RS_OVERLAP", "1" if world > 1 else "0"))
    dc.check(dc.lib.dc_model_set_option(st.model, b"rs_overlap", 0))
    step_no += 1
    rt.step(ranks, step_no, profile=1)
    dc.check(dc.lib.dc_model_set_option(st.model, b"rs_overlap", ov))
    ordered = rt.profile_json(st)
    barrier()
    tokens_box = world * T * n_micro
    value = tokens_box / (ms / 1e3)
    if offload_info:
        offload_info["pcie_gbs"] = offload_info["pcie_bytes_per_step"] / (ms / 1e3) / 1e9
        offload_info["pcie_frac_of_duplex"] = offload_info["pcie_gbs"] / offload_info["pcie_peak_gbs"]["duplex"]

    # ---- per-op breakdown of the last timed step (events recorded in-region)
    by = {}
    gemm_us, gemm_fl = 0, 0
    for o in last["ops"]:
        if o["kind"] in ("compute", "rs"):
            by.setdefault(o["name"], 0)
            by[o["name"]] += o["dur_us"]
            fl = gemm_flops(o["name"], cfg, T)
            if fl:
                gemm_us += o["dur_us"]
                gemm_fl += fl
    pk = peaks()
    achieved = gemm_fl / (gemm_us * 1e-6) / 1e12 if gemm_us else None
    ord_us = sum(o["dur_us"] for o in ordered["ops"] if o["kind"] == "compute" and gemm_flops(o["name"], cfg, T))
    traffic, traffic_note = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes_per_launch")
        traffic_note = "%s; algorithmic %s B" % (tj.get("launch"), tj.get("algorithmic_bytes_per_launch"))
        if tj.get("forward_launches_layer0"):
            traffic_note += "; DRAM / algorithmic per forward launch: " + ", ".join(
                "%s %.2fx" % (k, v["ratio"]) for k, v in tj["forward_launches_layer0"].items())
    except (OSError, ValueError):
        pass
    roofline = {"bound": "tensor", "kernel": "gemm2_bf16_sm100 (tcgen05 CTA pair, all layer GEMMs)",
                "achieved": achieved, "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16_tflops_sustained"] if achieved else None, "traffic": traffic,
                "traffic_note": traffic_note,
                "peak_source": pk["source"] + ", sustained bf16 (kernel inside a long step)",
                "flops_per_step": gemm_fl, "gemm_ms_per_step": gemm_us / 1e3,
                "achieved_stream_ordered": gemm_fl / (ord_us * 1e-6) / 1e12 if ord_us else None,
                "note": "achieved: GEMM op events of the last timed step (RS + Adam overlapped on its own stream: "
                        "a GEMM launched while rs_adam holds the SMs waits inside its events); "
                        "achieved_stream_ordered: one extra step with RS + Adam in compute-stream order"}
    shard_elems = st.layout.shard_elems
    rs_us = by.get("rs", 0)
    # per shard element: bf16 grads of N ranks + fp32 master/m/v r+w + bf16 shard w
    # (28 + 2(N-1) B at n = 1); with accumulation the first micro-step writes the
    # fp32 accumulator, the middle ones read+write it and the last one reads it
    per = 2 * world
    rs_bytes = ((per + 26) if n_micro == 1 else
                (per + 4) + (n_micro - 2) * (per + 8) + (per + 26 + 4)) * shard_elems
    kernels = {"op_ms_per_step": {k: round(v / 1e3, 3) for k, v in sorted(by.items())},
               "rs_adam": {"bytes_per_step": rs_bytes, "ms_per_step": rs_us / 1e3,
                           "achieved_gbs": rs_bytes / (rs_us * 1e-6) / 1e9 if rs_us else None,
                           "peak_gbs": pk["hbm_gbs"], "bound": "hbm" if world == 1 else "nvlink+hbm"}}

    # ---- end to end through the public API with HOST buffers: every step's
    # inputs cross PCIe from pinned memory inside the timed region, prefetched
    # one step ahead on a copy stream into a device staging buffer (as a data
    # loader would) and moved into the model's input buffers by a D2D copy at
    # the step's start; the loss is read back to the host after every step
    loss_host = torch.empty(n_micro, dtype=torch.float32).pin_memory()
    lp = rt.view(rt.loss_ptr(st), n_micro, torch.float32, device=dev)
    ps = torch.cuda.Stream(device=dev)
    x_stage, t_stage = torch.empty_like(x_dev), torch.empty_like(t_dev)
    ev_in, ev_used = torch.cuda.Event(), torch.cuda.Event()

    def h2d_prefetch():
        with torch.cuda.stream(ps):
            x_stage.view(-1).copy_(x_host, non_blocking=True)
            t_stage.view(-1).copy_(t_host, non_blocking=True)
            ev_in.record(ps)

    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    ps.wait_event(e0)
    h2d_prefetch()
    for k in range(args.steps):
        with torch.cuda.stream(cs):
            cs.wait_event(ev_in)
            x_dev.copy_(x_stage)
            t_dev.copy_(t_stage)
            ev_used.record(cs)
        if k + 1 < args.steps:
            ps.wait_event(ev_used)
            h2d_prefetch()
        step_no += 1
        one_step()
        with torch.cuda.stream(cs):
            loss_host.copy_(lp, non_blocking=True)
        cs.synchronize()
        _ = loss_host.tolist()
    dc.check(dc.lib.dc_model_join_states(st.model, cs.cuda_stream))
    e1.record(cs)
    barrier()
    ems = torch.tensor([e0.elapsed_time(e1) / args.steps], device=cdev)
    if world > 1:
        dist.all_reduce(ems, op=dist.ReduceOp.MAX, group=group)
    e2e = {"value": tokens_box / (ems.item() / 1e3), "unit": "tokens/s",
           "h2d_bytes_per_step": 2 * n_micro * T * cfg.hidden * 2, "d2h_bytes_per_step": 4 * n_micro,
           "loss": loss_host.tolist()[-1]}

    # ---- CPU oracle timed on host cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.model == "llama3-8b":
        sample_run = OracleSample(cfg, 128)
        t0 = time.perf_counter()
        for T in (32, 128, 32, 128):
            sample_run.step(T)
        val, a, b = sample_run.tokens_per_s(cfg)
        cpu = {"value": val, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": "1 Llama-3-8B-shaped layer at 32 and 128 tokens (2 samples each, %.1f s total), N=1: "
                         "oracle fwd+bwd+RS+Adam; t(T) = a + b T per layer, a = %.2f s, b = %.4f s/token, "
                         "extrapolated to %d layers x %d tokens" %
                         (time.perf_counter() - t0, a, b, cfg.layers, cfg.tokens)}

    # exposed communication (SURVEY §8 d): the compute stream's idle time in the
    # last timed step = step time - sum of compute-op events (each op's start
    # event is recorded after its waits on gathers / grad-slot flags)
    rs_in_order = int(os.environ.get("DC_RS_OVERLAP", "1" if world > 1 else "0")) == 0
    busy_ms = sum(o["dur_us"] for o in last["ops"]
                  if o["kind"] == "compute" or (rs_in_order and o["kind"] == "rs")) / 1e3
    # peak memory (SURVEY §8 d): every device buffer of the run is a torch
    # allocation (states, grad slots, flags, arena, activations, pool), so the
    # allocator's peak is the device total; the plan's own bound beside it
    mem = {"device_peak_allocated": torch.cuda.max_memory_allocated(dev),
           "device_peak_reserved": torch.cuda.max_memory_reserved(dev),
           "plan_peak": plan["peak_no_opt"] + plan.get("m_opt", 0) -
                         (offload_info["offloaded_bytes"] if offload_info else 0), "M": M}
    if offload_info:   # the reload ring is a static allocation beside the plan's live bytes
        mem["offload_pool"] = offload_info["pool_bytes"]
    mem["note"] = ("P_mem (a-3) is the executor's exact bookkeeping of its static allocations: bf16 shard + fp32 "
                   "master, grad slots, workspace, inputs, the saved activations live at each op and the gathered "
                   "buffers live under the schedule (m / v excluded, reading D14, added back as M_opt). " +
                   ("At N = 1 a gather aliases the shard, so the plan counts the gathered weights the device never "
                    "allocates (up to the bf16 weight bytes above the allocator's peak)." if world == 1 else
                    "At N > 1 the arena is one allocation of the plan's capacity, so the allocator's peak is the "
                    "plan's static part + arena capacity + every layer's activation buffer."))
    idle = {"ms": max(0.0, ms - busy_ms), "frac": max(0.0, ms - busy_ms) / ms,
            "note": "step time - compute-stream busy time of the last timed step (waits on gathers, "
                    "grad-slot / reduce-scatter flags and launch gaps; reduce-scatter ops count as busy when "
                    "they run in compute-stream order)"}
    if world > 1:
        exposed = dict(idle, target="< 10 % of the step (BASELINE north star)")
        if os.environ.get("DC_FUSED_AG", "0") not in ("", "0"):
            exposed["note"] += ("; fused_ag: a GEMM's waits for gather chunks fall inside its op events, so this "
                                "is a lower bound")
    else:
        exposed = {"ms": None, "frac": None, "note": "N = 1: no communication (gathers alias the shard, the "
                   "reduce-scatter reads only local grads); compute_stream_idle has the step's idle time"}
    coll = {"measured": False, "note": "N = 1: no collective runs; virtual-rank gather sweeps are in "
            "profiles/r02/ (scripts/ag_sweep.py)"}
    if world > 1:
        # per issued gather of the last timed step: transfer time (every receiver
        # ready -> every sender's stores landed here, CUDA events on the AG stream)
        dur = {o["id"]: o["dur_us"] for o in last["ops"] if o["kind"] == "ag"}
        ags = [(o["bytes"], dur.get(o["id"], 0)) for o in plan["ops"] if o["kind"] == "ag"]
        ags = [(b, us) for b, us in ags if us > 0]
        f = (world - 1) / world
        tot_b, tot_us = sum(b for b, _ in ags), sum(us for _, us in ags)
        big = [(b, us) for b, us in ags if b >= (64 << 20)]
        rs_per_layer_b = {}
        for p in last["params"]:
            rs_per_layer_b[p.get("layer", 0)] = rs_per_layer_b.get(p.get("layer", 0), 0) + p["bytes"]
        rs_us = [o["dur_us"] for o in last["ops"] if o["kind"] == "rs"]
        rs_b = sum(rs_per_layer_b.values())
        coll = {"measured": True, "n_ranks": dist.get_world_size(group),
                "transport": rt.symm_backend() if not args.share_gpu else "ipc (share-gpu test mode)",
                "note": "busbw = (N-1)/N x bytes / time; AG time from every receiver ready to all stores landed; "
                        "RS time = the fused reduce-scatter + Adam kernel (bf16 grads in over NVLink)",
                "gathers_per_step": len(ags), "ag_bytes_per_step": tot_b,
                "ag_busbw_gbs": f * tot_b / (tot_us * 1e-6) / 1e9 if tot_us else None,
                "ag_busbw_gbs_ge_64MiB": (f * sum(b for b, _ in big) / (sum(us for _, us in big) * 1e-6) / 1e9
                                          if big else None),
                "rs_busbw_gbs": f * rs_b / (sum(rs_us) * 1e-6) / 1e9 if rs_us and sum(rs_us) else None,
                "nvlink_peak_gbs": 900,
                "nvls": st.nvls or {"requested": 0, "note": "DC_NVLS=1|2|3 selects the multimem gather / "
                                    "ld_reduce reduce-scatter where the fabric gives multicast addresses"}}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": "%s-stack (%s): L=%d h=%d f=%d %d/%d heads%s, "
                                       "seq %d, b=%d per GPU, ZeRO-3 + proactive prefetch%s%s" %
                                       (args.model, MODELS[args.model][2], cfg.layers, cfg.hidden, cfg.ffn,
                                        cfg.n_heads, cfg.n_kv,
                                        ", %d experts top-2 (fixed balanced)" % cfg.n_experts if cfg.n_experts else "",
                                        args.seq, args.batch,
                                        " + selective unshard" if "S" in args.passes else "",
                                        (", grad accumulation %d" % n_micro if n_micro > 1 else "") +
                                        (", layer activation checkpointing" if args.checkpoint else "")),
                           "model": "%s-shaped synthetic stack (random init)" % args.model,
                           "global_batch": world * args.batch * n_micro, "micro_steps": n_micro,
                           "checkpoint": bool(args.checkpoint), "cuda_graph": bool(args.graph),
                           "seq_len": args.seq, "parallelism": "fsdp%d" % world, "passes": args.passes,
                           "mem_budget_M": M, "plan_ms": round(t_plan * 1e3, 2),
                           "unshard_params": len(plan["unshard"]), "offload": offload_info,
                           "tc_table": prof["tc"], "tc_source": tc_source, "tc_nccl_comparator": tc_nccl,
                           "fused_groups": sum(1 for o in plan["ops"] if o["kind"] == "ag" and
                                               len(o.get("members", [])) > 1),
                           "l2": "working set (~120 GB/GPU of weights, states, activations) >> 126 MB L2; no flush"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "exposed_comm": exposed, "compute_stream_idle": idle, "memory": mem,
                "clocks": clocks, "kernels": kernels, "collectives": coll,
                "host_enqueue_ms_per_step": round(host_enqueue_ms, 2)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
