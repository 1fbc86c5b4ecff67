mkdir -p gpurun_out scripts/_bin
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/attn_trace.cu $(ls build/csrc/*.o | grep -v attention_tc) -lcuda -o scripts/_bin/attn_trace > gpurun_out/r02aj_build.log 2>&1
for c in 0 200 290; do ./scripts/_bin/attn_trace 4 1024 16 f $c > gpurun_out/r02aj_attn_trace_cta$c.txt 2>&1; done
head -14 gpurun_out/r02aj_attn_trace_cta200.txt; tail -5 gpurun_out/r02aj_attn_trace_cta200.txt; tail -5 gpurun_out/r02aj_attn_trace_cta0.txt
timeout 300 python scripts/bench_attn.py scale > gpurun_out/r02aj_attn_scale.jsonl 2>&1
cat gpurun_out/r02aj_attn_scale.jsonl
