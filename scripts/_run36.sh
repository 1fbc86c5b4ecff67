mkdir -p gpurun_out
for t in 2 1; do
  CK_GEMM_STREAMK=$t timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/r02at_vs_cublas_sk$t.jsonl 2>&1
  echo "== streamk $t"; cat gpurun_out/r02at_vs_cublas_sk$t.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'shape' in d: print(d['shape'], d['ours_us'], d['cublas_us'])
    else: print(d)"
done
