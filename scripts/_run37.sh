mkdir -p gpurun_out
CK_GEMM_TILE=pair CK_GEMM_STREAMK=2 timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/r02au_vs_cublas.jsonl 2>&1
cat gpurun_out/r02au_vs_cublas.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'shape' in d: print(d['shape'], d['ours_us'], d['cublas_us'])
    else: print(d)"
