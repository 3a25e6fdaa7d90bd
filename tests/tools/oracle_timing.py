"""Oracle timing on the host cores ("Oracle timing"):

1. config 1 (4 x Linear(256, 256) MLP, fp32, 2 simulated ranks, b = 8 per
   rank): sharded step vs unsharded (replicated) step, seconds per step;
2. one synthetic Llama-3-8B-shaped layer at seq 256, 2 simulated ranks: the
   oracle's sharded step, tokens/s;
3. the oracle scheduler vs dc_plan (host-only C++) wall time on full-size S_0
   profiles of configs 2-5 (tests/sched_util.analytic_profile).

Each timed with BLAS threads = 1 and with all cores (the thread count is set
per child process, before numpy loads).  Prints one JSON object.

    python tests/tools/oracle_timing.py [--out profiles/r01g/oracle_timing.json]
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(item):
    sys.path.insert(0, ROOT)
    import dataclasses

    import synth
    from oracle import sched as osd
    from oracle import step as ost
    out = {}
    if item == "mlp":
        cfg = synth.MLP_CONFIG1
        table = synth.param_table(cfg)
        for name, mk, fn in (("sharded", lambda: ost.ShardedState(table, 2, bf16=False), ost.sharded_step),
                             ("unsharded", lambda: ost.ReplicatedState(table, 2, bf16=False), ost.replicated_step)):
            st = mk()
            fn(st, cfg, lr=1e-3)
            t0 = time.perf_counter()
            for _ in range(3):
                fn(st, cfg, lr=1e-3)
            out[name + "_s_per_step"] = (time.perf_counter() - t0) / 3
    elif item == "layer":
        cfg = dataclasses.replace(synth.LLAMA3_8B, layers=1, seq=256, batch=1)
        st = ost.ShardedState(synth.param_table(cfg), 2, bf16=True)
        t0 = time.perf_counter()
        ost.sharded_step(st, cfg, lr=1.5e-5)
        sec = time.perf_counter() - t0
        out = {"s_per_step": sec, "tokens_per_s": 2 * cfg.tokens / sec}
    elif item == "plan":
        from paper_2504_09983_b200 import dc
        from tests import sched_util as su
        op_ms = {"qkv": 0.3, "o_proj": 0.2, "gate_up": 0.7, "down": 0.35, "attn_norm": 0.02, "mlp_norm": 0.02,
                 "act": 0.05, "attn_mix": 0.03}
        cases = [("configs[1] llama3-8b L=32 N=8", "LLAMA3_8B", 32, 8, False, 155.7, osd.PASSES_PS),
                 ("configs[2] llama3-70b L=80 N=8 recompute M=130", "LLAMA3_70B", 80, 8, True, 130.0, osd.PASSES_PS),
                 ("configs[3] mixtral L=32 N=8", "MIXTRAL_8X7B", 32, 8, False, 155.7, osd.PASSES_PS),
                 ("configs[4] llama3-70b L=16 N=1 offload", "LLAMA3_70B", 16, 1, False, 165.6,
                  osd.PASSES_PS | osd.PASS_OFFLOAD | osd.PASS_HOST_STATES)]
        for label, name, L, N, ck, M_gb, passes in cases:
            cfg = dataclasses.replace(getattr(synth, name), layers=L, seq=2048, batch=1)
            prof, _, _, _ = su.analytic_profile(cfg, N, op_ms, checkpoint=ck)
            prof["tc"] = [[0, 20], [1 << 34, 20 + int((1 << 34) / 630e3)]]
            M = int(M_gb * 1e9)
            js = json.dumps(prof)
            t0 = time.perf_counter()
            o = osd.canonical_json(osd.plan(json.loads(js), M, passes=passes, strict=True))
            t_o = time.perf_counter() - t0
            t0 = time.perf_counter()
            h = dc.plan(js, M, passes=passes, strict=True)
            c = dc.schedule_json(h)
            t_c = time.perf_counter() - t0
            dc.lib.dc_schedule_free(h)
            out[label] = {"ops": len(prof["ops"]), "oracle_s": t_o, "dc_plan_s": t_c, "byte_identical": o == c}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--child", default="")
    args = ap.parse_args()
    if args.child:
        child(args.child)
        return
    cores = len(os.sched_getaffinity(0))
    res = {"cpu": platform.processor() or platform.machine(), "cores": cores}
    try:
        with open("/proc/cpuinfo") as f:
            res["cpu"] = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    for threads in (1, cores):
        env = dict(os.environ, OMP_NUM_THREADS=str(threads), OPENBLAS_NUM_THREADS=str(threads),
                   MKL_NUM_THREADS=str(threads))
        r = {}
        for item in ("mlp", "layer", "plan"):
            p = subprocess.run([sys.executable, __file__, "--child", item], capture_output=True, text=True, env=env,
                               cwd=ROOT, timeout=3600)
            r[item] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else {"error": p.stderr[-500:]}
        res["threads_%d" % threads] = r
    s = json.dumps(res, indent=1)
    print(s)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
