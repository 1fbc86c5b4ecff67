# r02ai: attention forward trace (clock-calibrated), ncu source-level stalls of the
# attention kernels, GEMM vs cuBLAS on the bench shapes
mkdir -p gpurun_out scripts/_bin
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/attn_trace.cu $(ls build/csrc/*.o | grep -v attention_tc) -lcuda -o scripts/_bin/attn_trace > gpurun_out/r02ai_build.log 2>&1
./scripts/_bin/attn_trace 4 1024 16 > gpurun_out/r02ai_attn_trace.txt 2>&1
head -16 gpurun_out/r02ai_attn_trace.txt; tail -4 gpurun_out/r02ai_attn_trace.txt
timeout 300 python scripts/attn_once.py > gpurun_out/r02ai_once.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_attn_.*_tc" -c 2 -o gpurun_out/r02ai_attn python scripts/attn_once.py > gpurun_out/r02ai_ncu.log 2>&1
echo "ncu rc=$?"
timeout 600 python scripts/gemm_vs_cublas.py > gpurun_out/r02ai_vs_cublas.jsonl 2>&1
tail -3 gpurun_out/r02ai_vs_cublas.jsonl
