O=gpurun_out/stack_fix
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532"
timeout 600 python -m pytest tests/test_stack_gpu.py tests/test_stack_local_gpu.py -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for g in cosine_topk noisy_topk sigmoid_topk expert_choice; do
  timeout 600 $TR tools/stack_on_box.py --config gpt2xl --gate $g --layers 4 --out $O > $O/stack_$g.log 2>&1
  echo "$g rc=$?"; tail -1 $O/stack_$g.log | cut -c1-400
done
