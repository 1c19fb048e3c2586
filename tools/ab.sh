#!/bin/bash
# Same-box A/B of two libfsmoe_cuda.so builds on the bench step: the current
# build vs _oldlib/libfsmoe_cuda_old.so (git-ignored; travels with gpurun).
# Alternates R bench runs of each (BENCH_ARGS, default the configs[2] step)
# and prints ms/step and the median SM clock of every run.
R=${R:-3}
ARGS=${BENCH_ARGS:-"--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-extra --no-timeline"}
L=paper_2501_10714_b200/lib
mkdir -p gpurun_out
cp $L/libfsmoe_cuda.so _oldlib/new.so
for r in $(seq 1 $R); do
  for v in new old; do
    if [ $v = new ]; then cp _oldlib/new.so $L/libfsmoe_cuda.so; else cp _oldlib/libfsmoe_cuda_old.so $L/libfsmoe_cuda.so; fi
    python bench.py $ARGS > gpurun_out/ab_${v}_$r.json 2> gpurun_out/ab_${v}_$r.err
    python - "$v" "$r" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], round(d["ms_per_step"], 3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"],
          round(d["roofline"]["frac"], 4))
except Exception as e:
    print(sys.argv[1], sys.argv[2], "failed", e)
PY
  done
done
cp _oldlib/new.so $L/libfsmoe_cuda.so
