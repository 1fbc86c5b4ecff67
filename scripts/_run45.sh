mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02bc_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02bc_smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02bc_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r02bc_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02bc_n1.json 2> gpurun_out/r02bc_n1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02bc_ref_n1.json 2> gpurun_out/r02bc_ref_n1.err; echo "ref rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/r02bc_n1.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'], d['clocks'], d['gpu_launches'], d['config']['stage_layers'])
r=json.loads(open('gpurun_out/r02bc_ref_n1.json').read().strip().splitlines()[-1])
print(r.get('value'), r.get('unit'), r.get('cpu_baseline',{}).get('sample','')[:200])"
