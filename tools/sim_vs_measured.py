"""schedule_sim's predicted fwd / bwd makespan (the planner's model, fitted on
the box) against the measured phase times of tools/sweep_on_box.py, per
transport; the regression view SURVEY §8f row 1 asks for.

    python tools/sim_vs_measured.py profiles/r01_sweep_p4.json
"""
import json
import statistics as st
import sys


def main(path):
    d = json.load(open(path))
    out = ["| transport | pass | measured / predicted: median | min | max | argmin simulated r == argmin measured r |",
           "|---|---|---|---|---|---|"]
    for tr in ("nccl", "peer"):
        for ps, i in (("fwd", 0), ("bwd", 1)):
            ratios, agree = [], 0
            for p in d["points"]:
                pred = {int(r): v[i] for r, v in p["predicted_ms"].items()}
                meas = {int(r): v[i] for r, v in p["measured_ms"][tr].items()}
                ratios += [meas[r] / pred[r] for r in pred]
                agree += min(pred, key=pred.get) == min(meas, key=meas.get)
            out.append(f"| {tr} | {ps} | {st.median(ratios):.2f} | {min(ratios):.2f} | {max(ratios):.2f} | "
                       f"{agree} / {len(d['points'])} |")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_sweep_p4.json")
