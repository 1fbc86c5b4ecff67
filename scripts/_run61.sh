# 8-GPU layout of configs[3] (one rank per process) as 8 processes on 4 GPUs, final build
mkdir -p gpurun_out
export NCCL_DEBUG=WARN CK_PROCS_PER_GPU=2
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 700 $TR --nproc-per-node 8 --master-port 29811 bench.py --gpus 8 --steps 10 --warmup 3 > gpurun_out/r02bo_cfg3_emu8.json 2> gpurun_out/r02bo_cfg3_emu8.err
echo "rc=$?"; grep "\[bench" gpurun_out/r02bo_cfg3_emu8.err | tail -3
python -c "
import json
d=json.loads(open('gpurun_out/r02bo_cfg3_emu8.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['ms_per_step'], d.get('diagnostics'), (d.get('bubble') or {}).get('measured'))"
