"""Per-kernel instruction counts of the main (largest backward-branch) loop in a cuobjdump -sass
listing: python scripts/sass_loops.py file.sass [name-filter] -- used to compare variants before
spending GPU time (integer address math, FP64 and load counts per layer iteration)."""
import collections
import re
import sys


def functions(path):
    cur, body = None, []
    for ln in open(path):
        m = re.search(r"Function : (\S+)", ln)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(ln)
    if cur:
        yield cur, body


def loop_mix(body):
    ins = []
    for ln in body:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), ln))
    best = None
    for a, op, ln in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", ln.split("BRA", 1)[1])
            if t and int(t.group(1), 16) < a and (best is None or a - int(t.group(1), 16) > best[1] - best[0]):
                best = (int(t.group(1), 16), a)
    if best is None:
        return None
    c = collections.Counter(op.split(".")[0] for a, op, _ in ins if best[0] <= a <= best[1])
    return c


if __name__ == "__main__":
    flt = sys.argv[2] if len(sys.argv) > 2 else ""
    for name, body in functions(sys.argv[1]):
        if flt not in name:
            continue
        c = loop_mix(body)
        if not c:
            continue
        tot = sum(c.values())
        fp = c["DFMA"] + c["DMUL"] + c["DADD"]
        it = c["IMAD"] + c["IADD3"] + c["LEA"] + c["SHF"] + c["VIADD"] + c["IADD"]
        ld = c["LDG"] + c["LDS"] + c["LDGSTS"] + c["LDL"]
        print(f"{name[:70]:70s} total {tot:5d} fp64 {fp:5d} int {it:4d} ld {ld:4d} st {c['STG'] + c['STS'] + c['STL']:3d} "
              f"spill {c['LDL'] + c['STL']}")
