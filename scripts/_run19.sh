mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py -m gpu -q --timeout 120 -x -k "stream_k" > gpurun_out/r02x_sk_tests.log 2>&1
echo "sk tests rc=$?"; tail -15 gpurun_out/r02x_sk_tests.log
timeout 600 python scripts/gemm_split_sweep.py > gpurun_out/r02x_sweep_sk.jsonl 2>&1
CK_GEMM_STREAMK=0 timeout 600 python scripts/gemm_split_sweep.py > gpurun_out/r02x_sweep_nosk.jsonl 2>&1
timeout 600 python scripts/gemm_wgrad_sweep.py > gpurun_out/r02x_wgrad_sk.jsonl 2>&1
python - <<'PY'
import json
a=[json.loads(l) for l in open('gpurun_out/r02x_sweep_sk.jsonl') if l.startswith('{')]
b=[json.loads(l) for l in open('gpurun_out/r02x_sweep_nosk.jsonl') if l.startswith('{')]
for x,y in zip(a,b): print(x['shape'], 'auto sk', x['auto'], 'no-sk', y['auto'])
for l in open('gpurun_out/r02x_wgrad_sk.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['shape'], 'auto', d['auto'], 'best', d['best'], d[d['best']] if d['best'] in d else '')
PY
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02x_b2.json 2> gpurun_out/r02x_b2.err
python -c "
import json
d=json.loads(open('gpurun_out/r02x_b2.json').read().strip().splitlines()[-1])
print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'], d['loss'])"
