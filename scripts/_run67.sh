mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for c in bert48 gpt2-medium; do
  i=$((i+1))
  timeout 400 $TR --nproc-per-node 4 --master-port 2983$i bench.py --gpus 4 --config $c --steps 10 --warmup 3 --diag-timeout 90 > gpurun_out/r02bu_$c.json 2> gpurun_out/r02bu_$c.err
  python -c "
import json
d=json.loads(open('gpurun_out/r02bu_$c.json').read().strip().splitlines()[-1])
print('$c', d['value'], d['ms_per_step'], d['config']['stage_layers'], (d.get('perfmodel') or {}).get('rel_err'))" 2>&1 | tail -1
done
