"""FP64 issue floor per kernel family from a --set full raw CSV export: executed DFMA + DMUL + DADD
warp instructions (the FP64 pipe issues 2 warp instructions per SM per cycle on B200: 64 FP64
lanes), the time they need at the pipe's peak at a given SM clock, and the kernel's measured
duration -- the share of the step the FP64 pipe alone accounts for.

    python scripts/fp64_floor.py profiles/r2_opt1_raw/full3d.csv [sm_mhz]
    python scripts/fp64_floor.py --json full3d.csv full2d.csv > profiles/<round>_fp64.json
          (FP64 warp instructions per launch of each bench.py timer key; bench.py reports the
           step's FP64 issue floor from the newest one)
"""
import csv
import sys

SMS = 148
PER_CLK = 2          # FP64 warp instructions per SM per cycle


def rows(path):
    r = list(csv.reader(open(path)))
    hdr, units = r[0], r[1]
    return hdr, units, [x for x in r[1:] if x and x[0].isdigit()]


def main(path, mhz=1750.0):
    hdr, units, data = rows(path)
    ix = {h: i for i, h in enumerate(hdr)}
    ops = ["smsp__sass_thread_inst_executed_op_%s_pred_on.sum.per_cycle_elapsed" % o for o in ("dfma", "dmul", "dadd")]
    seen = set()
    print(f"| kernel | ms (ncu) | FP64 warp inst | FP64 floor ms @ {mhz:.0f} MHz | floor / time |")
    print("|---|---:|---:|---:|---:|")
    for x in data:
        name = x[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        if name in seen:
            continue
        seen.add(name)
        cyc = float(x[ix["sm__cycles_elapsed.avg"]])
        per_cycle = sum(float(x[ix[o]]) for o in ops) / 32.0       # warp instructions per cycle, all SMSPs
        inst = per_cycle * cyc
        ms = float(x[ix["gpu__time_duration.sum"]]) * {"ms": 1.0, "us": 1e-3, "ns": 1e-6}[units[ix["gpu__time_duration.sum"]]]
        floor = inst / (SMS * PER_CLK) / (mhz * 1e3)
        print(f"| `{name}` | {ms:.3f} | {inst:.3e} | {floor:.3f} | {floor / ms:.2f} |")


def per_key(paths):
    """bench.py timer key -> FP64 warp instructions per launch (first captured launch of each kernel)."""
    sys.path.insert(0, __import__("os").path.dirname(__file__))
    from traffic_json import KEYS
    inst = {}
    for path in paths:
        hdr, units, data = rows(path)
        ix = {h: i for i, h in enumerate(hdr)}
        ops = ["smsp__sass_thread_inst_executed_op_%s_pred_on.sum.per_cycle_elapsed" % o for o in ("dfma", "dmul", "dadd")]
        for x in data:
            name = x[ix["Kernel Name"]].split("(")[0].replace("void ", "")
            if name not in inst:
                inst[name] = sum(float(x[ix[o]]) for o in ops) / 32.0 * float(x[ix["sm__cycles_elapsed.avg"]])
    out = {}
    for key, prefixes in KEYS.items():
        got = [n for pre in prefixes for n in inst if n.startswith(pre)][:len(prefixes)]
        if len(got) == len(prefixes):
            out[key] = {"fp64_warp_inst": sum(inst[n] for n in got), "kernel": " + ".join(got), "source": paths[0]}
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--json":
        import json
        print(json.dumps(per_key(sys.argv[2:]), indent=1))
    else:
        main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1750.0)
