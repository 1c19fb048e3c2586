"""Markdown table of a tools/sweep_on_box.py JSON (planner vs measured best,
the online refinement bench.py uses)."""
import json
import sys


def main(path):
    d = json.load(open(path))
    pts = d["points"]
    ok_ref = sum(1 for p in pts if p["best_step"]["refined_over_best"] <= 1.05)
    ok_plan = sum(1 for p in pts if p["best_step"]["plan_peer_over_best"] <= 1.05)
    out = [f"Wall {d['wall_s']:.0f} s, {d['world']} GPUs. Refined choice within 5 % of the measured best "
           f"(transport x r): {ok_ref} / {len(pts)}; the analytic plan alone (peer transport at the planned r): "
           f"{ok_plan} / {len(pts)}.", "",
           "| T | M | E | k | planned r (fwd, bwd) | best (transport, r) | best ms | refined (transport, r) | "
           "refined / best | plan / best |", "|---|---|---|---|---|---|---|---|---|---|"]
    for p in pts:
        b = p["best_step"]
        out.append(f"| {p['T']} | {p['M']} | {p['E']} | {p['k']} | {p['plan']['r_fwd']}, {p['plan']['r_bwd']} | "
                   f"{b['transport']}, {b['r']} | {b['ms']:.3f} | {p['refined']['transport']}, {p['refined']['r']} | "
                   f"{b['refined_over_best']:.3f} | {b['plan_peer_over_best']:.3f} |")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
