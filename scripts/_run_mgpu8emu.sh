# The 8-GPU layout of configs[3] (one logical rank per process, every stage message
# remote, 2-holder NCCL stage communicators) as 8 processes on 4 GPUs (2 per GPU):
# a path check of what the driver's 8-GPU run executes.
mkdir -p gpurun_out
export NCCL_DEBUG=WARN CK_PROCS_PER_GPU=2
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 8 --master-port 29571 bench.py --gpus 8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ac_cfg3_emu8.json 2> gpurun_out/r02ac_cfg3_emu8.err
echo "rc=$?"; grep "\[bench" gpurun_out/r02ac_cfg3_emu8.err | tail -3
python -c "
import json
d=json.loads(open('gpurun_out/r02ac_cfg3_emu8.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['bubble'], d['perfmodel']['rel_err'], d['sync_policies'], d['loss'], d['gpu_launches'])"
