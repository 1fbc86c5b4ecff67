mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for e in "CK_NCCL_MAX_CTAS=0" "CUDA_DEVICE_MAX_CONNECTIONS=8" "X=1" "CK_NCCL_MAX_CTAS=0 CK_GEMM_STREAMK=0"; do
  i=$((i+1))
  env $e timeout 600 $TR --nproc-per-node 4 --master-port 2976$i bench.py --gpus 4 --config q4 --steps 10 --warmup 3 --no-cpu-baseline --diag-timeout 120 > gpurun_out/r02bi_$i.json 2> gpurun_out/r02bi_$i.err
  python -c "
import json
d=json.loads(open('gpurun_out/r02bi_$i.json').read().strip().splitlines()[-1])
print('$e', d['value'], d['ms_per_step'], {k: v['ms_per_step'] for k, v in (d.get('sync_policies') or {}).items()}, d.get('comm'))" 2>&1 | tail -1
done
