# final multi-GPU validation (uncapped NCCL CTAs): configs[3] on 4 and 2 GPUs, 4-process parity
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
show() { python -c "
import json
d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['value'], d['e2e']['value'], d['ms_per_step'], d.get('diagnostics'), (d.get('perfmodel') or {}).get('rel_err'), {k: v['ms_per_step'] for k, v in (d.get('sync_policies') or {}).items()})" 2>&1 | tail -1; }
timeout 900 $TR --nproc-per-node 4 --master-port 29781 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02bk_cfg3_n4.json 2> gpurun_out/r02bk_cfg3_n4.err
echo "n4 rc=$?"; show gpurun_out/r02bk_cfg3_n4.json
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29782 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02bk_cfg3_n2.json 2> gpurun_out/r02bk_cfg3_n2.err
echo "n2 rc=$?"; show gpurun_out/r02bk_cfg3_n2.json
for o in sgd adamw zero; do MP_OPT=$o timeout 300 $TR --nproc-per-node 4 --master-port 2979$((RANDOM%9)) scripts/mp_check.py >> gpurun_out/r02bk_mp_check.jsonl 2>> gpurun_out/r02bk_mp_check.err; echo "mp $o rc=$?"; done
grep -c world gpurun_out/r02bk_mp_check.jsonl
