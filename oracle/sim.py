"""Three-stream timing replay of a planned schedule.  TEST INFRASTRUCTURE ONLY.

Used to pin Algorithm 1 against the paper's overlap claim (Fig. 5, PAPER.md
lines 258-266: without prefetching "all-gather operations are issued just
before computation, resulting in no overlap") and SPEC S:390-391.

Streams: compute (compute ops, releases), comm (gathers, reduce-scatters),
copy (offload/reload).  Issue semantics (reading D23): a gather scheduled at
position i cannot start before the compute-stream op preceding position i in
the schedule has finished — this is what makes S_0 serial (Fig. 5a).  A
compute op starts after every gather holding one of its params has finished.
Times are exact Fractions of µs.
"""
from fractions import Fraction

from .sched import tc_eval


def simulate(plan_ops, prof, copy_us_per_byte=Fraction(0)):
    s0 = prof["ops"]
    B = {p["id"]: p["bytes"] for p in prof["params"]}
    tc = [tuple(x) for x in prof["tc"]]
    ready = {"compute": Fraction(0), "comm": Fraction(0), "copy": Fraction(0)}
    last_compute_end = Fraction(0)
    holder_end = {}        # param -> end time of the latest gather holding it
    end = Fraction(0)
    for e in plan_ops:
        k = e["kind"]
        if k in ("compute", "rel"):
            start = ready["compute"]
            if k == "compute":
                for p in s0[e["id"]]["params"]:
                    start = max(start, holder_end.get(p, Fraction(0)))
                dur = Fraction(s0[e["id"]]["dur_us"])
            else:
                dur = Fraction(0)
            ready["compute"] = start + dur
            last_compute_end = ready["compute"]
            end = max(end, ready["compute"])
        elif k in ("ag", "rs"):
            start = max(ready["comm"], last_compute_end)
            if k == "ag":
                dur = tc_eval(tc, sum(B[p] for p in e["members"]))
            else:
                dur = Fraction(s0[e["id"]]["dur_us"])
            ready["comm"] = start + dur
            if k == "ag":
                for p in e["members"]:
                    holder_end[p] = ready["comm"]
            end = max(end, ready["comm"])
        else:
            start = max(ready["copy"], last_compute_end)
            ready["copy"] = start + copy_us_per_byte * e["bytes"]
            end = max(end, ready["copy"])
    return end
