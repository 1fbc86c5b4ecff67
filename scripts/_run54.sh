mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for spec in "X=1:" "X=1:--head-efficiency 1.0" "CK_GEMM_STREAMK=0:" "X=1:--partition even"; do
  e=${spec%%:*}; a=${spec#*:}; i=$((i+1))
  env $e timeout 600 $TR --nproc-per-node 4 --master-port 2975$i bench.py --gpus 4 --config q4 --steps 10 --warmup 3 --no-cpu-baseline --diag-timeout 120 $a > gpurun_out/r02bh_$i.json 2> gpurun_out/r02bh_$i.err
  python -c "
import json
d=json.loads(open('gpurun_out/r02bh_$i.json').read().strip().splitlines()[-1])
print('$spec', d['value'], d['ms_per_step'], d['config']['stage_layers'], {k: v['ms_per_step'] for k, v in (d.get('sync_policies') or {}).items()})" 2>&1 | tail -1
done
