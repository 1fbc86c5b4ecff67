mkdir -p gpurun_out/timelines
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
show() { python -c "
import json,sys
d=json.loads(open('$1').read().strip().splitlines()[-1])
b=d['bubble']
print('$1', d['value'], d['ms_per_step'], d['config']['stage_layers'], 'bubble', b['measured'], b['measured_per_rank'], 'ref@B/F', b['reference_schedule_at_measured_B/F'], b['measured_B/F'], 'dessim', b['dessim_at_measured_profile'], 'eq1', d['perfmodel']['rel_err'])" 2>&1 | tail -1; }
i=0
for spec in "gpt2-medium-d4:X=1" "gpt2-1.3b-d4:CK_BWD_FUSE=0" "gpt2-1.3b-d4:X=1" "gpt2-medium-d4-n8fd:CK_BWD_FUSE=0"; do
  c=${spec%%:*}; e=${spec#*:}; i=$((i+1))
  env $e CK_TIMELINE=gpurun_out/timelines/r02az_$c$i timeout 420 $TR --nproc-per-node 4 --master-port 2970$i bench.py --gpus 4 --config $c --steps 20 --warmup 5 > gpurun_out/r02az_$c$i.json 2> gpurun_out/r02az_$c$i.err
  echo "$c $e rc=$?"; show gpurun_out/r02az_$c$i.json
done
