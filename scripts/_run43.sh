mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for spec in "gpt2-medium-d4:0.67" "gpt2-medium-d4:1.0" "gpt2-medium-d4:0.67" "gpt2-medium-d4:1.0" "gpt2-1.3b-d4:0.67" "gpt2-1.3b-d4:1.0" "gpt2-1.3b-d4:0.67" "gpt2-1.3b-d4:1.0"; do
  c=${spec%%:*}; h=${spec#*:}; i=$((i+1))
  timeout 420 $TR --nproc-per-node 4 --master-port 2971$i bench.py --gpus 4 --config $c --steps 20 --warmup 5 --head-efficiency $h --diag-timeout 200 > gpurun_out/r02ba_$i.json 2> gpurun_out/r02ba_$i.err
  python -c "
import json
d=json.loads(open('gpurun_out/r02ba_$i.json').read().strip().splitlines()[-1])
b=d.get('bubble') or {}
print('$c head=$h', d['value'], d['ms_per_step'], d['config']['stage_layers'], b.get('measured'), b.get('reference_schedule_at_measured_B/F'))" 2>&1 | tail -1
done
