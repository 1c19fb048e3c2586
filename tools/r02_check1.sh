#!/bin/bash
# 1-GPU check: the whole -m gpu suite, the tile-order DRAM probe, and the
# configs[2] GEMM ncu capture with the current build.
mkdir -p gpurun_out/c1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/c1/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/c1/gpu_tests.log
python tools/order_probe.py > /dev/null 2>&1 || echo "order probe failed (no ncu)"
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c1/order.csv python tools/order_probe.py > gpurun_out/c1/order_ncu.log 2>&1
echo "order ncu rc=$?"
python tools/order_probe.py --summarise gpurun_out/c1/order.csv > gpurun_out/c1/order.md 2>&1; tail -60 gpurun_out/c1/order.md
CFG=mixtral bash tools/profile_r02.sh > gpurun_out/c1/prof.log 2>&1; echo "prof rc=$?"
