mkdir -p gpurun_out scripts/_bin
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/gemm_trace.cu $(ls build/csrc/*.o | grep -v cuda_gemm) -lcuda -o scripts/_bin/gemm_trace > gpurun_out/r02aw_build.log 2>&1
for c in 96 98 100; do CK_GEMM_TILE=pair CK_GEMM_STREAMK=2 ./scripts/_bin/gemm_trace 2528 1280 5120 0 0 0 $c; done
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -k "stream_k" 2>&1 | tail -2
CK_GEMM_TILE=pair CK_GEMM_STREAMK=2 timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/r02aw_vs_cublas.jsonl 2>&1
cat gpurun_out/r02aw_vs_cublas.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'shape' in d: print(d['shape'], d['ours_us'], d['cublas_us'])
    else: print(d)"
