mkdir -p gpurun_out
for c in 8 32 8 32; do
CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bm_c$c.json 2> gpurun_out/r02bm_c$c.err
python -c "
import json
d=json.loads(open('gpurun_out/r02bm_c$c.json').read().strip().splitlines()[-1])
print('conn=$c', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
