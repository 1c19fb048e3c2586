#!/bin/bash
# Gate kernels: routing / noise parity tests, same-box A/B against
# _oldlib/libfsmoe_cuda_old.so, and ncu captures of screen_tc / exact_final at
# both shapes (configs[1]: launches 0-1, configs[2]: launch 4 of tools/gate_probe.py).
O=gpurun_out/gate_ncu
mkdir -p $O
python -m pytest tests/test_routing_gpu.py tests/test_noise_exact_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -2
R=${R:-2} bash tools/gate_ab.sh 2>&1 | grep -E "pruned|shape"
for k in screen_tc exact_final; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/${k}_c1 -f python tools/gate_probe.py 1 > $O/ncu_${k}_c1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o $O/${k}_c2 -f python tools/gate_probe.py 1 > $O/ncu_${k}_c2.log 2>&1
  echo "$k ncu rc=$?"
done
