#!/bin/bash
# Round-2 multi-GPU session (run under gpurun --gpus N): EP / stack tests on
# real GPUs, the bench at N over transports and pipeline degrees, and the
# configs[4] gradient-partition stack for every gate.
N=${N:-4}
O=gpurun_out/multi_p$N
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
timeout 1200 python -m pytest tests/test_ep_gpu.py tests/test_stack_gpu.py tests/test_stack_local_gpu.py -q -x > $O/tests.log 2>&1
echo "tests rc=$?"; tail -3 $O/tests.log
for cfg in gpt2m mixtral; do
  steps=50; [ $cfg = mixtral ] && steps=10
  for tr in peer ce; do
    for r in 1 2 4; do
      [ $tr = peer ] && [ $r != 1 ] && [ $cfg = mixtral ] && continue
      FSMOE_EP_TRANSPORT=$tr timeout 600 $TR bench.py --gpus $N --config $cfg --r-fwd $r --r-bwd $r \
        --steps $steps --warmup 3 --no-e2e --no-extra --warm-seconds 2 > $O/bench_${cfg}_${tr}_r$r.json 2> $O/bench_${cfg}_${tr}_r$r.err
      python - $O/bench_${cfg}_${tr}_r$r.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ex = d.get("exposed_alltoall") or {}
    print(sys.argv[1].split("/")[-1], round(d["ms_per_step"], 3), round(d["value"] / 1e6, 3), "Mtok/s",
          "exposed", round(ex.get("ms_per_step", 0), 3), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"],
          "frac", round(d["step_roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
    done
  done
done
for g in noisy_topk sigmoid_topk cosine_topk expert_choice; do
  timeout 600 $TR tools/stack_on_box.py --config gpt2xl --gate $g --layers 4 --out $O > $O/stack_$g.log 2>&1
  tail -1 $O/stack_$g.log
done
