#!/bin/bash
# End-of-round multi-GPU evidence on one 4-GPU box: EP / stack tests, the
# default bench at N = 2 and 4 (online pipeline choice), and the configs[4]
# gradient-partition stack for every gate.
O=gpurun_out/multi_final
mkdir -p $O
timeout 1500 python -m pytest tests/test_ep_gpu.py tests/test_stack_gpu.py tests/test_stack_local_gpu.py tests/test_ep_local_gpu.py -q > $O/tests.log 2>&1
echo "tests rc=$?"; tail -2 $O/tests.log
for n in 2 4; do
  devs=$(seq -s, 0 $((n-1)))
  CUDA_VISIBLE_DEVICES=$devs timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 20 --warmup 5 > $O/bench_n$n.json 2> $O/bench_n$n.err
  echo "bench n=$n rc=$?"
  python - $O/bench_n$n.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"] / 1e6, 4), "Mtok/s", round(d["ms_per_step"], 3), "ms", d["clocks"]["sm_mhz"],
      d["config"]["pipeline"].get("chosen"), "exposed", d["exposed_alltoall"]["by_rank_ms_per_step"],
      "e2e", round(d["e2e"]["value"] / 1e6, 4), "frac", round(d["step_roofline"]["frac"], 3),
      "c1", round(d["configs[1]"]["value"] / 1e6, 3))
PY
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
for g in noisy_topk sigmoid_topk cosine_topk expert_choice; do
  timeout 600 $TR tools/stack_on_box.py --config gpt2xl --gate $g --layers 4 --out $O > $O/stack_$g.log 2>&1
  tail -1 $O/stack_$g.log | cut -c1-400
done
