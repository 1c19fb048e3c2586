#!/bin/bash
# ncu DRAM bytes + duration of every launch of one bench step (configs[2] and
# configs[1]), summarised per kernel with achieved HBM GB/s (tools/route_hbm.py).
O=gpurun_out/route_hbm
mkdir -p $O
for cfg in mixtral gpt2m; do
  CMD="python bench.py --config $cfg --steps 2 --warmup 3 --warm-seconds 0 --no-e2e --no-cpu-baseline --no-extra --no-timeline"
  $CMD > $O/plain_$cfg.json 2> $O/plain_$cfg.err || { echo "$cfg bench failed"; continue; }
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -c 400 \
      --csv --log-file $O/$cfg.csv $CMD > $O/ncu_$cfg.log 2>&1
  echo "$cfg ncu rc=$?"
  python tools/route_hbm.py $O/$cfg.csv
done
