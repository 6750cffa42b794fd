"""DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of each stepper kernel family
from a --set full raw CSV export -> profiles/<round>_traffic.json (bench.py reports it as roofline.traffic).

    python scripts/traffic_json.py profiles/r1_opt3_raw/full3d.csv profiles/r1_opt3_raw/full2d.csv > profiles/r1_traffic.json
"""
import csv
import json
import sys

# bench.py timer name -> kernel-name prefixes whose (first captured) launches make up that call
KEYS = {
    "r": ["k_compute_r_t<1"],
    "project": ["k_project<0"],
    "f3d2d": ["k_hrhs_t<2, 1"],
    "wtilde": ["k_compute_wtilde_t"],
    "rhs_uT_s1": ["k_hrhs_s<3, 2, 1, 1"],     # stage 1 (u = u0, T = T0)
    "rhs_uT_s2": ["k_hrhs_s<3, 2, 1, 0"],
    "vertical_u_impl": ["k_vimpl_fwd<2", "k_vimpl_bwd_r<2"],
    "vertical_T_impl": ["k_vimpl_fwd<1", "k_vimpl_bwd_r<1"],
    "vertical_u_expl": ["k_vexpl3<2"],
    "vertical_T_expl": ["k_vexpl3<1"],
    "rk_stage0": ["k_rk_stage<0"],
    "rk_stage1": ["k_rk_stage<1"],
    "rk_stage2": ["k_rk_stage<2"],
}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def rows(path):
    r = list(csv.reader(open(path)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        name = row[hdr.index("Kernel Name")].replace("void ", "").replace("pdg::", "")
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            b += float(row[i]) * UNIT[units[i]]
        yield name, b


if __name__ == "__main__":
    first = {}
    src = {}
    for p in sys.argv[1:]:
        for name, b in rows(p):
            for key, prefs in KEYS.items():
                for pre in prefs:
                    if name.startswith(pre) and (key, pre) not in first:
                        first[(key, pre)] = (name, b)
                        src[key] = p
    out = {}
    for key, prefs in KEYS.items():
        if all((key, p) in first for p in prefs):
            out[key] = {"kernel": " + ".join(first[(key, p)][0].split("(")[0] for p in prefs),
                        "dram_bytes": sum(first[(key, p)][1] for p in prefs), "source": src[key]}
    print(json.dumps(out, indent=1))
