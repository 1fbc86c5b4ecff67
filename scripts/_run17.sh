mkdir -p gpurun_out scripts/_bin
make -s -j16 -C paper_2107_06925_b200/csrc > /dev/null 2>&1
for P in 0 2 3 4; do
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -DCK_ATTN_POLY_EVERY=$P -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/attn_trace.cu $(ls build/csrc/*.o | grep -v attention_tc) -lcuda -o scripts/_bin/attn_trace_p$P > /dev/null 2>&1
echo "poly every $P: $(./scripts/_bin/attn_trace_p$P 4 1024 16 | grep 'avg launch')  s632: $(./scripts/_bin/attn_trace_p$P 4 632 20 | grep 'avg launch')"
done
