#!/bin/bash
# Bitwise checks + L2-hint DRAM probe + gate A/B (round 2).
mkdir -p gpurun_out/l2hint
python tools/gemm_determinism.py 16 48 80 144 > gpurun_out/l2hint/det_c1.log 2>&1; tail -1 gpurun_out/l2hint/det_c1.log
python tools/gemm_determinism.py 16 48 80 144 --mixtral > gpurun_out/l2hint/det_mix.log 2>&1; tail -1 gpurun_out/l2hint/det_mix.log
python -m pytest tests/test_routing_gpu.py tests/test_noise_exact_gpu.py -x -q 2>&1 | tail -2
bash tools/gate_ab.sh 2>&1 | grep -E "pruned|shape" > gpurun_out/l2hint/gate_ab.log; cat gpurun_out/l2hint/gate_ab.log
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l2hint/l2hint.csv python tools/l2hint_probe.py > gpurun_out/l2hint/ncu.log 2>&1
python tools/l2hint_probe.py --summarise gpurun_out/l2hint/l2hint.csv
