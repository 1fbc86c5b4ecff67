mkdir -p gpurun_out/timelines
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CK_TIMELINE=gpurun_out/timelines/r02_13bd4 timeout 600 $TR --nproc-per-node 4 --master-port 29581 bench.py --gpus 4 --config gpt2-1.3b-d4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ae_13bd4_n4.json 2> gpurun_out/r02ae_a.err
echo "rc=$?"; grep "\[bench" gpurun_out/r02ae_a.err | tail -2
timeout 600 $TR --nproc-per-node 4 --master-port 29582 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ae_cfg3_n4.json 2> gpurun_out/r02ae_b.err
echo "rc=$?"; grep "\[bench" gpurun_out/r02ae_b.err | tail -2
for f in gpurun_out/r02ae_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d['value'], d['ms_per_step'], d['bubble'], d['perfmodel']['rel_err'], d['sync_policies'])"; done
