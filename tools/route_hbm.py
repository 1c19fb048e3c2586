"""Achieved HBM bandwidth of every non-GEMM kernel of one step (routing,
permutations, gate, gate backward) from an ncu CSV with
dram__bytes_read.sum, dram__bytes_write.sum and gpu__time_duration.sum
(one launch per row group), against MEASURED_PEAKS.json's copy bandwidth.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none -c 400 --csv --log-file OUT.csv python bench.py ...
    python tools/route_hbm.py OUT.csv [first-kernel-of-a-step] [steps-to-skip]

ncu runs each kernel alone with cold caches (its default cache control), so
these are standalone DRAM figures: bytes are what the kernel itself moves.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def main(path, marker="w_prep_kernel", skip=3):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    ii, ki, mi, vi, ui = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"),
                          h.index("Metric Value"), h.index("Metric Unit"))
    per, names = {}, {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        i = int(r[ii])
        names[i] = r[ki].split("(")[0].replace("void ", "").replace("fsmoe::<unnamed>::", "")
        per.setdefault(i, {})[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    ids = sorted(per)
    starts = [i for i in ids if marker in names[i]]
    s0 = starts[skip]
    s1 = starts[skip + 1] if len(starts) > skip + 1 else ids[-1] + 1
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6547.8) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6547.8
    out = []
    lines = [f"| kernel | us | DRAM read MB | DRAM write MB | achieved GB/s | of {peak:.0f} GB/s |",
             "|---|---|---|---|---|---|"]
    for i in ids:
        if i < s0 or i >= s1:
            continue
        m = per[i]
        t = m.get("gpu__time_duration.sum", 0.0)
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        gbs = (rd + wr) / t / 1e9 if t > 0 else 0.0
        out.append({"kernel": names[i], "us": t * 1e6, "read_mb": rd / 1e6, "write_mb": wr / 1e6, "gbs": gbs,
                    "frac": gbs / peak})
        lines.append(f"| {names[i][:44]} | {t * 1e6:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {gbs:.0f} | "
                     f"{gbs / peak:.2f} |")
    print("\n".join(lines))
    with open(os.path.splitext(path)[0] + ".json", "w") as f:
        json.dump({"peak_gbs": peak, "launches": out}, f, indent=1)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], a[1] if len(a) > 1 else "w_prep_kernel", int(a[2]) if len(a) > 2 else 3)
