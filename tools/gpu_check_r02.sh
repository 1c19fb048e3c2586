set -x
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv) > gpurun_out/host.txt 2>&1
timeout 900 python -m pytest tests/test_ep_local_gpu.py -x -q > gpurun_out/local_ep.log 2>&1; echo "local_ep rc=$?"
tail -5 gpurun_out/local_ep.log
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_ep_local_gpu.py > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_default.json
tail -5 gpurun_out/bench_default.err
