mkdir -p gpurun_out
for r in 0 23; do
CK_GEMM_RATE192=$r timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ax_r$r.json 2> gpurun_out/r02ax_r$r.err
python -c "
import json
d=json.loads(open('gpurun_out/r02ax_r$r.json').read().strip().splitlines()[-1])
print('rate192=$r', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['frac'])"
done
