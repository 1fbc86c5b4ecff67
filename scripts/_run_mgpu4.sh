# 4 GPUs, one process per GPU.  D=4 W=1 configs: one logical rank per GPU -> measured bubble,
# valid Eq.-1 prediction, sync-policy A/B; configs[3] with 2 ranks per GPU; 2-GPU line.
mkdir -p gpurun_out/timelines
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CK_TIMELINE=gpurun_out/timelines/r02_d4n8bh timeout 900 $TR --nproc-per-node 4 --master-port 29511 bench.py --gpus 4 --config gpt2-medium-d4-n8bh --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_d4n8bh_n4.json 2> gpurun_out/r02e_d4n8bh_n4.err
CK_TIMELINE=gpurun_out/timelines/r02_d4n4 timeout 900 $TR --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 --config gpt2-medium-d4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_d4n4_n4.json 2> gpurun_out/r02e_d4n4_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29513 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_cfg3_n4.json 2> gpurun_out/r02e_cfg3_n4.err
timeout 900 $TR --nproc-per-node 2 --master-port 29514 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_cfg3_n2.json 2> gpurun_out/r02e_cfg3_n2.err
for f in gpurun_out/r02e_*.json; do echo $f; tail -c 1500 $f; echo; done
tail -5 gpurun_out/r02e_*.err
