mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02be_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r02be_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02be_n1.json 2> gpurun_out/r02be_n1.err; echo "bench rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/r02be_n1.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'], d['clocks'])"
