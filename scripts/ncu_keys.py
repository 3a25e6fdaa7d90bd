"""Per-launch key metrics of ncu --set full reports (memory-bound kernels):
time, DRAM bytes and throughput, L2 / L1 traffic, occupancy, issue activity,
registers.  Usage: ncu_keys.py rep1.ncu-rep [rep2 ...] > table.md"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem % peak"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__cycles_elapsed.avg.per_second", "SM clk"), ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long-sb"),
        ("lts__t_bytes.sum", "L2 bytes")]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units, rows = r[0], r[1], r[2:]
    cols = [(h.index(k), lab) for k, lab in KEYS if k in h]
    ik = h.index("Kernel Name")
    print("\n#### %s\n" % rep.split("/")[-1])
    print("| # | kernel | " + " | ".join("%s (%s)" % (lab, units[j]) for j, lab in cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    for i, row in enumerate(rows):
        print("| %d | %s | %s |" % (i, row[ik].split("(")[0].replace("void ", ""), " | ".join(row[j] for j, _ in cols)))
