mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for r in 23 0 23 0; do
  i=$((i+1))
  CK_GEMM_RATE192=$r timeout 420 $TR --nproc-per-node 4 --master-port 2972$i bench.py --gpus 4 --config gpt2-1.3b-d4 --steps 20 --warmup 5 --diag-timeout 200 > gpurun_out/r02bb_$i.json 2> gpurun_out/r02bb_$i.err
  python -c "
import json
d=json.loads(open('gpurun_out/r02bb_$i.json').read().strip().splitlines()[-1])
print('13bd4 rate192=$r', d['value'], d['ms_per_step'], (d.get('bubble') or {}).get('measured'))" 2>&1 | tail -1
done
