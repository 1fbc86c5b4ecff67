mkdir -p gpurun_out scripts/_bin
for P in 3 2 4 0; do
nvcc -std=c++20 -O3 -DCK_ATTN_POLY_EVERY=$P -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/attn_trace.cu $(ls build/csrc/*.o | grep -v attention_tc) -lcuda -o scripts/_bin/attn_trace_p$P > /dev/null 2>&1
for B in 4 16; do echo "poly_every=$P B=$B $(./scripts/_bin/attn_trace_p$P $B 1024 16 f 0 | grep 'avg launch')"; done
done
