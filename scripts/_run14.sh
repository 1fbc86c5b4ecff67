mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02s_b2.json 2> gpurun_out/r02s_b2.err
python -c "
import json
d=json.loads(open('gpurun_out/r02s_b2.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'])"
bash scripts/_run_ncu.sh
