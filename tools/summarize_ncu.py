"""Summaries of ncu outputs for profiles/: launch-list shares and key metrics
of --set full captures.  Usage: python tools/summarize_ncu.py launches.csv [rep...]"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print(f"kernel launches: {sum(a[0] for a in agg.values())}, total device time {tot:.2f} ms")
    print(f"{'ms':>9} {'share':>6} {'n':>5}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
        print(f"{t:9.3f} {100 * t / tot:5.1f}% {c:5d}  {k}")


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    print(f"== {rep}")
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print("kernel:", name[:100])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k} = {v[i]} {u[i]}")


if __name__ == "__main__":
    launches(sys.argv[1])
    for rep in sys.argv[2:]:
        full(rep)
