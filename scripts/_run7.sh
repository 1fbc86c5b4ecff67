mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpt_gpu.py tests/test_gpt_wide_gpu.py -m gpu -q --timeout 600 > gpurun_out/r02h_tests.log 2>&1
tail -5 gpurun_out/r02h_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_b2.json 2> gpurun_out/r02h_b2.err
CK_BWD_FUSE=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_b2_nobwdfuse.json 2> gpurun_out/r02h_b2_nobwdfuse.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --B 1 > gpurun_out/r02h_b1.json 2> gpurun_out/r02h_b1.err
for f in gpurun_out/r02h_*.json; do python -c "
import json,sys
try:
  d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'], d['loss'])
except Exception as e: print('$f', 'ERR', e)"; done
tail -3 gpurun_out/r02h_b2.err
