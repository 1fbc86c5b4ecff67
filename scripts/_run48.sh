# final-build multi-GPU lines: configs[3] on 2 and 4 GPUs (the driver's scaling commands), default flags
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
show() { python -c "
import json
d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['value'], d['e2e']['value'], d['ms_per_step'], d['clocks'], d.get('diagnostics'), (d.get('perfmodel') or {}).get('rel_err'), {k: v['ms_per_step'] for k, v in (d.get('sync_policies') or {}).items()})" 2>&1 | tail -1; }
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29731 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02bd_cfg3_n2.json 2> gpurun_out/r02bd_cfg3_n2.err
echo "n2 rc=$?"; show gpurun_out/r02bd_cfg3_n2.json
timeout 900 $TR --nproc-per-node 4 --master-port 29732 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02bd_cfg3_n4.json 2> gpurun_out/r02bd_cfg3_n4.err
echo "n4 rc=$?"; show gpurun_out/r02bd_cfg3_n4.json
timeout 900 $TR --nproc-per-node 4 --master-port 29733 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02bd_ref_n4.json 2> gpurun_out/r02bd_ref_n4.err
echo "ref n4 rc=$?"; tail -c 300 gpurun_out/r02bd_ref_n4.json
