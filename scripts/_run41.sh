mkdir -p gpurun_out
for r in 1 0 1 0; do
CK_GEMM_STREAMK=$r timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ay_sk$r.json 2> gpurun_out/r02ay_sk$r.err
python -c "
import json
d=json.loads(open('gpurun_out/r02ay_sk$r.json').read().strip().splitlines()[-1])
print('streamk=$r', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['frac'])"
done
