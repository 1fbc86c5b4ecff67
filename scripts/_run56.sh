mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for spec in "gpt2-1.3b:CK_NCCL_MAX_CTAS=0" "gpt2-1.3b:CK_NCCL_MAX_CTAS=16" "gpt2-1.3b-d4:CK_NCCL_MAX_CTAS=0" "gpt2-1.3b-d4:CK_NCCL_MAX_CTAS=16"; do
  c=${spec%%:*}; e=${spec#*:}; i=$((i+1))
  env $e timeout 600 $TR --nproc-per-node 4 --master-port 2977$i bench.py --gpus 4 --config $c --steps 10 --warmup 3 --no-cpu-baseline --diag-timeout 150 > gpurun_out/r02bj_$i.json 2> gpurun_out/r02bj_$i.err
  python -c "
import json
d=json.loads(open('gpurun_out/r02bj_$i.json').read().strip().splitlines()[-1])
print('$spec', d['value'], d['ms_per_step'], {k: v['ms_per_step'] for k, v in (d.get('sync_policies') or {}).items()})" 2>&1 | tail -1
done
