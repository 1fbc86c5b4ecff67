mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for c in q4 q4-gpipe q4-dapple; do
  i=$((i+1))
  timeout 600 $TR --nproc-per-node 4 --master-port 2980$i bench.py --gpus 4 --config $c --steps 10 --warmup 3 --no-cpu-baseline --diag-timeout 120 > gpurun_out/r02bl_$c.json 2> gpurun_out/r02bl_$c.err
  python -c "
import json
d=json.loads(open('gpurun_out/r02bl_$c.json').read().strip().splitlines()[-1])
print('$c', d['value'], d['ms_per_step'], (d.get('perfmodel') or {}).get('rel_err'))" 2>&1 | tail -1
done
