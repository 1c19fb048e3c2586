#!/bin/bash
# Round-2 profile capture on the GPU box (repo root), configs[2] (the
# default bench workload) unless CFG is set:
#   1. the bench command without ncu (must exit 0 first),
#   2. the per-launch list of the same command (gpu__time_duration.sum),
#   3. --set full of one step's GEMM launches: the gate screen's, the six expert GEMMs, the gate backward's.
set -u
CFG=${CFG:-mixtral}
OUT=gpurun_out/prof_$CFG
mkdir -p $OUT
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --warm-seconds 0 --no-e2e --no-cpu-baseline --no-extra --no-timeline"
$CMD > $OUT/bench_plain.json 2> $OUT/bench_plain.err || { echo "bench failed"; tail -20 $OUT/bench_plain.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    $CMD > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
# grouped_gemm launches per step: the gate screen, the six expert GEMMs and, for a
# top-k > 1 softmax gate, the gate backward's two (x^T G and the in-place dx)
PER=$([ "$CFG" = mixtral ] && echo 9 || echo 7)
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s $((3 * PER)) -c $PER \
    -o $OUT/gemm_full -f $CMD > $OUT/ncu_gemm.log 2>&1
echo "gemm full rc=$?"
ls -la $OUT
