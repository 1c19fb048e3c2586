"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per step."""
import collections
import csv
import sys


def main(path, marker="rowdot", skip_steps=3):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    seq = []
    for r in rows[hi + 1:]:
        if len(r) > vi:
            seq.append((r[ki].split("(")[0].replace("fsmoe::<unnamed>::", "").replace("void ", "")[:48],
                        float(r[vi].replace(",", "")) / 1000.0))
    starts = [i for i, (n, _) in enumerate(seq) if marker in n]
    s0, s1 = starts[skip_steps], starts[skip_steps + 1]
    step = seq[s0:s1]
    tot = sum(v for _, v in step)
    agg = collections.defaultdict(float)
    for n, v in step:
        agg[n] += v
    print(f"one step: {len(step)} launches, {tot:.1f} us (ncu serialised, cold-ish)")
    for n, v in step:
        print(f"  {v:8.1f} us  {100*v/tot:5.1f}%  {n}")
    print("by kernel:")
    for n, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"  {v:8.1f} us  {100*v/tot:5.1f}%  {n}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], a[1] if len(a) > 1 else "rowdot", int(a[2]) if len(a) > 2 else 3)
