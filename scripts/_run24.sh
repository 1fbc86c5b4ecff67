mkdir -p gpurun_out scripts/_bin
make -s -j16 -C paper_2107_06925_b200/csrc > /dev/null 2>&1
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/attn_trace.cu $(ls build/csrc/*.o | grep -v attention_tc) -lcuda -o scripts/_bin/attn_trace > /dev/null 2>&1
./scripts/_bin/attn_trace 4 1024 16 > gpurun_out/r02ad_attn_trace.txt 2>&1
head -14 gpurun_out/r02ad_attn_trace.txt
timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/r02ad_vs_cublas.jsonl 2>&1
cat gpurun_out/r02ad_vs_cublas.jsonl
