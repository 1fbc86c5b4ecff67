mkdir -p gpurun_out scripts/_bin
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/gemm_trace.cu $(ls build/csrc/*.o | grep -v cuda_gemm) -lcuda -o scripts/_bin/gemm_trace > gpurun_out/r02av_build.log 2>&1
for c in 0 40 100 146; do CK_GEMM_TILE=pair CK_GEMM_STREAMK=2 ./scripts/_bin/gemm_trace 2528 1280 5120 0 0 0 $c; done
CK_GEMM_TILE=pair CK_GEMM_STREAMK=0 ./scripts/_bin/gemm_trace 2528 1280 5120 0 0 0 0
