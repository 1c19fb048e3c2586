#!/bin/bash
# ncu --set full of the gate's tensor-core screen (screen GEMM + screen_tc)
# and exact_final at the configs[1] and configs[2] shapes (tools/gate_probe.py).
O=gpurun_out/gate_ncu
mkdir -p $O
python tools/gate_probe.py 1 > $O/probe.log 2>&1 || { echo probe failed; tail $O/probe.log; exit 1; }
for k in screen_tc_kernel exact_final_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 4 -o $O/$k -f python tools/gate_probe.py 1 > $O/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -c 1 -o $O/screen_gemm -f python tools/gate_probe.py 1 > $O/ncu_screen_gemm.log 2>&1
echo "screen_gemm rc=$?"
