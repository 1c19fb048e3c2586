#!/bin/bash
# Regenerates tests/golden/planio/*.golden.json from the reference planner
# (oracle/_ref/plan_tool, built from /root/reference by `make -C oracle plan_tool`).
# Inputs (bench CSV measured on the box, the two model files) are ours.
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
G=$HERE/../tests/golden/planio
T=$HERE/_ref/plan_tool
make -s -C "$HERE" plan_tool
$T fit "$G/bench_p4.csv" 0 > "$G/fit_p4.golden.json"
python3 - "$G" <<'PY'
import json, sys
g = sys.argv[1]
d = json.load(open(f"{g}/fit_p4.golden.json"))
d.pop("fit")
open(f"{g}/profile_p4.json", "w").write(json.dumps(d, indent=2) + "\n")
PY
for m in box4 multinode; do
  $T plan "$G/model_$m.json" "$G/profile_p4.json" > "$G/plan_$m.golden.json"
  for style in fsmoe pipemoe; do
    for pass in fwd bwd; do
      $T simulate "$G/model_$m.json" "$G/profile_p4.json" $style $pass 1 > "$G/sim_${m}_${style}_${pass}.golden.json"
    done
  done
done
