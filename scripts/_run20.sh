mkdir -p gpurun_out
CK_GEMM_STREAMK=0 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err
echo "bench rc=$?"; tail -12 gpurun_out/r02y_bench.err
python -c "
import json
d=json.loads(open('gpurun_out/r02y_bench.json').read().strip().splitlines()[-1])
print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'], d['cpu_baseline'])" 2>&1 | tail -2
