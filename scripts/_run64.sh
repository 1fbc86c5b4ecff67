mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_gpt_gpu.py -x -q 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02br_n1.json 2> gpurun_out/r02br_n1.err; echo "bench rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/r02br_n1.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'], d['clocks'])"
