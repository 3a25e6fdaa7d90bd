"""Summarise a round's ncu artifacts (scripts/profile_round.sh) into markdown:
launch-list shares per kernel, and per-launch key metrics of the --set full
captures.  Usage: summarize_profiles.py <prof_dir> [launch csv] [capture names...] > summary.md"""
import collections
import csv
import io
import subprocess
import sys

d = sys.argv[1]


def launches(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.reader(io.StringIO("".join(lines)))
    h = next(r)
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    iu = h.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
    for row in r:
        if row[im] == "gpu__time_duration.sum":
            rows.append((row[ik], float(row[iv].replace(",", "")) * scale.get(row[iu], 1.0)))
    return rows


rows = launches(d + "/" + (sys.argv[2] if len(sys.argv) > 2 else "launches.csv"))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for k, v in rows:
    k = k.split("(")[0] if not k.startswith("void") else k.split("(")[0]
    tot[k] += v
    cnt[k] += 1
S = sum(tot.values())
print("| kernel | launches | total us | share |\n|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print("| %s | %d | %.1f | %.1f %% |" % (k.strip(), cnt[k], v, 100 * v / S))


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


KEYS = [("gpu__time_duration.sum", "time"), ("sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active", "tcgen05 %"),
        ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor-mem %"),
        ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("sm__cycles_elapsed.avg.per_second", "SM clk"), ("launch__registers_per_thread", "regs")]
for name in (sys.argv[3:] or ["gemm2", "rs_adam"]):
    try:
        h, units, rows = raw("%s/%s.ncu-rep" % (d, name))
    except Exception as e:
        print("\n(%s: %s)" % (name, e))
        continue
    print("\n### ncu --set full: %s\n" % name)
    cols = [(h.index(k), lab) for k, lab in KEYS if k in h]
    print("| # | kernel | grid | " + " | ".join("%s (%s)" % (lab, units[j]) for j, lab in cols) + " |")
    print("|---|---|---|" + "---|" * len(cols))
    ig = h.index("launch__grid_size") if "launch__grid_size" in h else None
    ik = h.index("Kernel Name")
    for i, r in enumerate(rows):
        print("| %d | %s | %s | %s |" % (i, r[ik].split("(")[0], r[ig] if ig is not None else "",
                                        " | ".join(r[j] for j, _ in cols)))
