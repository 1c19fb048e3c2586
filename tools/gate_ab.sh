#!/bin/bash
# Same-box A/B of the gate (tools/gate_probe.py, 20 reps per path) between
# the current libfsmoe_cuda.so and _oldlib/libfsmoe_cuda_old.so.
R=${R:-3}
L=paper_2501_10714_b200/lib
cp $L/libfsmoe_cuda.so _oldlib/new.so
for r in $(seq 1 $R); do
  for v in new old; do
    if [ $v = new ]; then cp _oldlib/new.so $L/libfsmoe_cuda.so; else cp _oldlib/libfsmoe_cuda_old.so $L/libfsmoe_cuda.so; fi
    python tools/gate_probe.py 20 2>&1 | grep -E "shape|us per gate" | sed "s/^/$v $r: /"
  done
done
cp _oldlib/new.so $L/libfsmoe_cuda.so
