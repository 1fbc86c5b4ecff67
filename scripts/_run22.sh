mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py -m gpu -q --timeout 600 -k "stream_k" > gpurun_out/r02aa_sk_tests.log 2>&1
echo "sk tests rc=$?"; tail -4 gpurun_out/r02aa_sk_tests.log
timeout 600 python scripts/gemm_wgrad_sweep.py > gpurun_out/r02aa_wgrad.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02aa_wgrad.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['shape'], 'auto', d['auto'], d['auto_tflops'], 'best', d['best'], d[d['best']] if d['best'] in d else '')
PY
for i in 1 2; do
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02aa_bench$i.json 2> gpurun_out/r02aa_bench$i.err
echo "bench$i rc=$?"; tail -3 gpurun_out/r02aa_bench$i.err
python -c "
import json
d=json.loads(open('gpurun_out/r02aa_bench$i.json').read().strip().splitlines()[-1])
print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'], d['e2e']['value'])"
done
