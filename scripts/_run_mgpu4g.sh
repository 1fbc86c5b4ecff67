# r02ah: 13bd4 timeline on 4 GPUs, 8-process emulation with issue trace + diag watchdog, N=1 line
mkdir -p gpurun_out/timelines
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
show() { python -c "
import json,sys
d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['value'], d['e2e']['value'], d['ms_per_step'], (d.get('bubble') or {}).get('measured'), (d.get('perfmodel') or {}).get('rel_err'), d.get('diagnostics'), d.get('gpu_launches'))" 2>&1 | tail -1; }
CK_TIMELINE=gpurun_out/timelines/r02ah_13bd4 timeout 420 $TR --nproc-per-node 4 --master-port 29631 bench.py --gpus 4 --config gpt2-1.3b-d4 --steps 20 --warmup 5 > gpurun_out/r02ah_13bd4_n4.json 2> gpurun_out/r02ah_13bd4_n4.err
echo "13bd4 n4 rc=$? $(grep '\[bench' gpurun_out/r02ah_13bd4_n4.err | tail -1)"; show gpurun_out/r02ah_13bd4_n4.json
CK_TRACE_ISSUE=2 CK_PROCS_PER_GPU=2 timeout 500 $TR --nproc-per-node 8 --master-port 29641 bench.py --gpus 8 --steps 10 --warmup 3 --diag-timeout 150 > gpurun_out/r02ah_cfg3_emu8.json 2> gpurun_out/r02ah_cfg3_emu8.err
echo "emu8 rc=$? $(grep '\[bench' gpurun_out/r02ah_cfg3_emu8.err | tail -1)"; show gpurun_out/r02ah_cfg3_emu8.json
grep "iteration issued" gpurun_out/r02ah_cfg3_emu8.err | tail -12
for p in 0 1 2 3 4 5 6 7; do grep "\[issue\] proc $p " gpurun_out/r02ah_cfg3_emu8.err | tail -1; done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02ah_n1.json 2> gpurun_out/r02ah_n1.err
echo "n1 rc=$?"; show gpurun_out/r02ah_n1.json
