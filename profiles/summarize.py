"""Summarise ncu outputs into profiles/<round>_summary.md.

    python profiles/summarize.py <launches.csv> <full.ncu-rep> <out.md>

launches.csv: `ncu --metrics gpu__time_duration.sum --csv --log-file` of one
bench command (cold-cache, serialised launches: compare SHARES).
full.ncu-rep: `ncu --set full` capture of the same command's key kernels.
"""
import csv
import subprocess
import sys
from collections import OrderedDict


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "").split("<")[0]
        name = name.split("::")[-1]
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    return agg


METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
        vals = []
        for key, label in METRICS:
            cands = [i for i, k in enumerate(h) if k == key] + \
                    [i for i, k in enumerate(h) if k.endswith("." + key) and r[i].strip()]
            if cands:
                i = cands[0]
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("n/a")
        res.append((name, vals))
    return res


def main():
    launches, rep, out = sys.argv[1:4]
    lines = ["# ncu summary", "",
             f"Launch list: `{launches}` (ncu `gpu__time_duration.sum`, cold-cache, serialised).",
             "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    agg = launch_shares(launches)
    tot = sum(v[1] for v in agg.values())
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
    lines += ["", f"Full capture: `{rep}` (`ncu --set full`).", "",
              "| kernel | " + " | ".join(l for _, l in METRICS) + " |",
              "|---|" + "---|" * len(METRICS)]
    for name, vals in full_metrics(rep):
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
