# multi-process validation after the stage-collective rendezvous (r02ag)
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
show() { python -c "
import json,sys
d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['value'], d['e2e']['value'], d['ms_per_step'], d['bubble'].get('measured'), d['perfmodel']['rel_err'], {k: v['ms_per_step'] for k, v in (d.get('sync_policies') or {}).items()})" 2>&1 | tail -1; }
for i in 1 2; do
  timeout 420 $TR --nproc-per-node 4 --master-port 2961$i bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ag_cfg3_n4_$i.json 2> gpurun_out/r02ag_cfg3_n4_$i.err
  echo "cfg3 n4 #$i rc=$? $(grep '\[bench' gpurun_out/r02ag_cfg3_n4_$i.err | tail -1)"; show gpurun_out/r02ag_cfg3_n4_$i.json
done
CUDA_VISIBLE_DEVICES=0,1 timeout 420 $TR --nproc-per-node 2 --master-port 29621 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ag_cfg3_n2.json 2> gpurun_out/r02ag_cfg3_n2.err
echo "cfg3 n2 rc=$? $(grep '\[bench' gpurun_out/r02ag_cfg3_n2.err | tail -1)"; show gpurun_out/r02ag_cfg3_n2.json
CK_TIMELINE=gpurun_out/timelines/r02ag_13bd4 timeout 420 $TR --nproc-per-node 4 --master-port 29631 bench.py --gpus 4 --config gpt2-1.3b-d4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ag_13bd4_n4.json 2> gpurun_out/r02ag_13bd4_n4.err
echo "13bd4 n4 rc=$? $(grep '\[bench' gpurun_out/r02ag_13bd4_n4.err | tail -1)"; show gpurun_out/r02ag_13bd4_n4.json
CK_PROCS_PER_GPU=2 timeout 600 $TR --nproc-per-node 8 --master-port 29641 bench.py --gpus 8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ag_cfg3_emu8.json 2> gpurun_out/r02ag_cfg3_emu8.err
echo "emu8 rc=$? $(grep '\[bench' gpurun_out/r02ag_cfg3_emu8.err | tail -1)"; show gpurun_out/r02ag_cfg3_emu8.json
for o in sgd adamw zero; do MP_OPT=$o timeout 300 $TR --nproc-per-node 4 --master-port 2965$((RANDOM%9)) scripts/mp_check.py >> gpurun_out/r02ag_mp_check.jsonl 2>> gpurun_out/r02ag_mp_check.err; echo "mp $o rc=$?"; done
tail -3 gpurun_out/r02ag_mp_check.jsonl
