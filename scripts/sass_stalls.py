"""Top stall sites of an ncu --page source --print-source sass CSV export: for each of the N
instructions with the most samples of a stall reason, the instruction and the producer of its
first source register (the load or spill the warp is waiting on)."""
import csv
import re
import sys


def main(path, reason="stall_long_sb", n=12):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    hdr = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
    v = lambda x: int(x) if x.isdigit() else 0  # noqa: E731
    col = hdr.index(reason)
    tot = sum(v(r[col]) for r in data)
    allc = hdr.index("Warp Stall Sampling (All Samples)")
    print(f"{reason}: {tot} of {sum(v(r[allc]) for r in data)} samples")
    top = sorted(range(len(data)), key=lambda i: -v(data[i][col]))[:n]
    for i in sorted(top):
        ins = data[i][1].strip()
        regs = re.findall(r"\bR(\d+)\b", ins.split(",", 1)[1] if "," in ins else "")
        prod = ""
        for r in regs:
            for j in range(i - 1, max(0, i - 400), -1):
                dst = re.match(r"\s*(?:@!?P\d+\s+)?[A-Z][A-Z0-9_.]*\s+R(\d+)", data[j][1])
                if dst and dst.group(1) == r and re.search(r"\b(LD|LDL|LDG|LDS|LDGSTS)", data[j][1]):
                    prod = f"  <- [{j}] {data[j][1].strip()[:60]}"
                    break
            if prod:
                break
        print(f"{i:5d} {v(data[i][col]):7d}  {ins[:60]}{prod}")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3] or []))
