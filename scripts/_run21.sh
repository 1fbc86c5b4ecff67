mkdir -p gpurun_out scripts/_bin
make -s -j16 -C paper_2107_06925_b200/csrc > /dev/null 2>&1
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/gemm_trace.cu $(ls build/csrc/*.o | grep -v cuda_gemm) -lcuda -o scripts/_bin/gemm_trace > gpurun_out/r02z_build.log 2>&1
for blk in 0 2 4; do ./scripts/_bin/gemm_trace 2528 1280 1280 0 0 0 $blk; done > gpurun_out/r02z_trace.txt 2>&1
CK_GEMM_STREAMK=0 ./scripts/_bin/gemm_trace 2528 1280 1280 0 0 0 0 >> gpurun_out/r02z_trace.txt 2>&1
cat gpurun_out/r02z_trace.txt; tail -3 gpurun_out/r02z_build.log
