"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and a --set full report.

    python scripts/ncu_summary.py gpurun_out/launches.csv gpurun_out/prof.ncu-rep > profiles/<name>.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("sass__inst_executed_local_loads", "local ld"),
]


def short(name):
    return name.split("(")[0].replace("void ", "")


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    unit = None
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1.0)
        a = agg[short(r[ik])]
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {t:.3f} | {100 * t / tot:.1f}% |")
    out.append(f"| **sum** | {sum(a[0] for a in agg.values())} | {tot:.3f} | 100% |")
    return "\n".join(out)


HEADER = [True]


def full(path):
    if path.endswith(".csv"):
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m, _ in METRICS if m in hdr}
    ik = hdr.index("Kernel Name")
    cols = [lbl for m, lbl in METRICS if m in idx]
    out = ["| kernel | " + " | ".join(cols) + " |", "|---" * (len(cols) + 1) + "|"] if HEADER[0] else []
    HEADER[0] = False
    for r in rows[2:]:
        vals = []
        for m, _ in METRICS:
            if m in idx:
                v, u = r[idx[m]], units[idx[m]]
                try:
                    v = f"{float(v):.4g}"
                except ValueError:
                    pass
                vals.append(v + (f" {u}" if u and u not in ("%", "inst", "warp", "register/thread") else ""))
        out.append(f"| `{short(r[ik])}` | " + " | ".join(vals) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    print("## Launch list (ncu gpu__time_duration, --clock-control none; cold-cache, serialised)\n")
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print("\n## --set full capture (one launch per kernel family)\n")
        for p in sys.argv[2:]:
            print(full(p))
