mkdir -p gpurun_out/p4ab
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513"
$TR bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/p4ab/default.json 2> gpurun_out/p4ab/default.err; echo default rc=$?
for i in 1 2; do
 for v in "peer 1" "ce 2" "ce 3"; do set -- $v
  $TR bench.py --gpus 4 --steps 20 --warmup 3 --transport $1 --r-fwd $2 --r-bwd $2 --no-e2e --no-extra --no-cpu-baseline --no-timeline > gpurun_out/p4ab/${1}_r$2_$i.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/p4ab/${1}_r$2_$i.json').read().strip().splitlines()[-1]); print('$1 r$2 $i', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['exposed_alltoall']['by_rank_ms_per_step'])"
 done
done
