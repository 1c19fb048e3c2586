#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   1. the bench command without ncu (must exit 0 first),
#   2. the per-launch list of the same command (ncu, gpu__time_duration.sum),
#   3. --set full of one step's six expert GEMM launches and of the gate's
#      dominant kernel, with source correlation.
# Outputs under gpurun_out/prof/; summaries are copied into profiles/.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $OUT/bench_plain.log 2>&1 || { echo "bench failed"; tail -20 $OUT/bench_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    $CMD > $OUT/ncu_launch.log 2>&1
# launches per step: skip the 3 warm-up steps of GEMMs (6 each)
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 18 -c 6 \
    -o $OUT/gemm_full -f $CMD > $OUT/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:screen_kernel -s 3 -c 1 \
    -o $OUT/gate_full -f $CMD > $OUT/ncu_gate.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dispatch_bulk_kernel -s 3 -c 1 \
    -o $OUT/dispatch_full -f $CMD > $OUT/ncu_dispatch.log 2>&1
ls -la $OUT
