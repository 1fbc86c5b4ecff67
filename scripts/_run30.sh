mkdir -p gpurun_out scripts/_bin
timeout 600 python -m pytest tests/test_ops_gpu.py -x -q -k attention > gpurun_out/r02ao_attn_tests.log 2>&1; echo "attn tests rc=$?"; tail -2 gpurun_out/r02ao_attn_tests.log
timeout 300 python scripts/bench_attn.py > gpurun_out/r02ao_attn.jsonl 2>&1; cat gpurun_out/r02ao_attn.jsonl
for R in 0 1; do
nvcc -std=c++20 -O3 -DCK_ATTN_DQ_RED=$R -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/attn_trace.cu $(ls build/csrc/*.o | grep -v attention_tc) -lcuda -o scripts/_bin/attn_trace$R > gpurun_out/r02ao_build.log 2>&1
./scripts/_bin/attn_trace$R 4 1024 16 b 0 > gpurun_out/r02ao_bwd_trace_red$R.txt 2>&1
echo "red=$R: $(grep 'avg launch' gpurun_out/r02ao_bwd_trace_red$R.txt)"
done
head -12 gpurun_out/r02ao_bwd_trace_red1.txt
