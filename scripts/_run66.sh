mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python bench.py > gpurun_out/r02bt_n1.json 2> gpurun_out/r02bt_n1.err; echo "bench n1 rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/r02bt_n1.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['config'], d['cpu_baseline']['value'] if d['cpu_baseline'] else None, d['gpu_launches'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29821 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02bt_n2.json 2> gpurun_out/r02bt_n2.err; echo "bench n2 rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/r02bt_n2.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['config']['parallelism'], d.get('diagnostics'))"
