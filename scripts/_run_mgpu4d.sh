mkdir -p gpurun_out/timelines
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CK_BWD_FUSE=0 CK_TIMELINE=gpurun_out/timelines/r02_d4n8fd_nobwdfuse_graph timeout 900 $TR --nproc-per-node 4 --master-port 29561 bench.py --gpus 4 --config gpt2-medium-d4-n8fd --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_d4n8fd_nobwdfuse_n4.json 2> gpurun_out/r02p_a.err
CK_TIMELINE=gpurun_out/timelines/r02_d4n4_graph timeout 900 $TR --nproc-per-node 4 --master-port 29562 bench.py --gpus 4 --config gpt2-medium-d4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_d4n4_n4.json 2> gpurun_out/r02p_b.err
timeout 900 $TR --nproc-per-node 4 --master-port 29563 bench.py --gpus 4 --config gpt2-1.3b-d4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_13bd4_n4.json 2> gpurun_out/r02p_c.err
CK_BWD_FUSE=0 timeout 900 $TR --nproc-per-node 4 --master-port 29564 bench.py --gpus 4 --config gpt2-1.3b-d4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_13bd4_nobwdfuse_n4.json 2> gpurun_out/r02p_d.err
for f in gpurun_out/r02p_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d['value'], d['ms_per_step'], d['bubble']['measured'], d['bubble']['reference_schedule_at_measured_B/F'], d['bubble']['dessim_at_measured_profile'], d['perfmodel']['rel_err'], d['mfu']['frac_of_sustained'])"; done
