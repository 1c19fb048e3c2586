#!/bin/bash
# Same-box A/B of programmatic dependent launch (FSMOE_PDL=1 default vs 0) on
# the bench step: configs[1] (launch-bound boundaries matter most) and configs[2].
O=gpurun_out/pdl_ab
mkdir -p $O
for r in 1 2 3; do
  for v in 1 0; do
    for cfg in gpt2m mixtral; do
      FSMOE_PDL=$v python bench.py --config $cfg --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extra \
        > $O/${cfg}_pdl${v}_$r.json 2> $O/${cfg}_pdl${v}_$r.err
      python - "$O/${cfg}_pdl${v}_$r.json" "$cfg" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "pdl", sys.argv[3], round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[2], "pdl", sys.argv[3], "failed", e)
PY
    done
  done
done
