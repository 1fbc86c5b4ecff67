mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/r02ar_gemm_tests.log 2>&1; echo "gemm tests rc=$?"; tail -3 gpurun_out/r02ar_gemm_tests.log
for t in pair pair192 default; do
  if [ $t = default ]; then timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/r02ar_vs_cublas_$t.jsonl 2>&1
  else CK_GEMM_TILE=$t timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/r02ar_vs_cublas_$t.jsonl 2>&1; fi
  echo "== $t"; cat gpurun_out/r02ar_vs_cublas_$t.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'shape' in d: print(d['shape'], d['ours_us'], d['cublas_us'])
    else: print(d)"
done
