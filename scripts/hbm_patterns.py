"""HBM bandwidth of the traffic patterns the virtual-rank gathers produce, for
context of their "fraction of the copy peak" (MEASURED_PEAKS.json hbm_gbs is
a 1:1 read:write copy): device-to-device copy (1 read : 1 write), memset
(write only) and one source written to N destinations with cudaMemcpyAsync
(1 read : N writes, the ag_push pattern at N virtual ranks).  CUDA events,
median of 5 after 2 warm-ups.  One JSON line."""
import json
import statistics

import torch


def timed(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return statistics.median(ts)


def main():
    n = 1 << 30
    src = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {}
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    t = timed(lambda: dst.copy_(src))
    out["copy_1to1_gbs"] = 2 * n / t / 1e9
    t = timed(lambda: dst.fill_(7))
    out["memset_gbs"] = n / t / 1e9
    for N in (2, 8):
        m = n // N
        dsts = [torch.empty(m, dtype=torch.uint8, device="cuda") for _ in range(N)]
        s = src[:m]
        t = timed(lambda: [d.copy_(s) for d in dsts])
        out["one_to_%d_gbs" % N] = (m * N + m * N) / t / 1e9      # each copy reads its source once
        out["one_to_%d_read1_write%d_gbs" % (N, N)] = (m + m * N) / t / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
