mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r02i_tests.log 2>&1
tail -8 gpurun_out/r02i_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_b2.json 2> gpurun_out/r02i_b2.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --B 1 > gpurun_out/r02i_b1.json 2> gpurun_out/r02i_b1.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config gpt2-medium > gpurun_out/r02i_medium.json 2> gpurun_out/r02i_medium.err
for f in gpurun_out/r02i_*.json; do python -c "
import json,sys
try:
  d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'], d['loss'])
except Exception as e: print('$f', 'ERR', e)"; done
