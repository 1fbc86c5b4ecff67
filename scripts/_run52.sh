mkdir -p gpurun_out
for r in 1 0 1 0; do
CK_STREAM_PRIO=$r timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bf_p$r.json 2> gpurun_out/r02bf_p$r.err
python -c "
import json
d=json.loads(open('gpurun_out/r02bf_p$r.json').read().strip().splitlines()[-1])
print('prio=$r', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
