mkdir -p gpurun_out scripts/_bin
timeout 600 python -m pytest tests/test_ops_gpu.py -x -q -k attention > gpurun_out/r02al_attn_tests.log 2>&1; echo "attn tests rc=$?"; tail -3 gpurun_out/r02al_attn_tests.log
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/attn_trace.cu $(ls build/csrc/*.o | grep -v attention_tc) -lcuda -o scripts/_bin/attn_trace > gpurun_out/r02al_build.log 2>&1
./scripts/_bin/attn_trace 4 1024 16 b 0 > gpurun_out/r02al_bwd_trace_cta0.txt 2>&1
./scripts/_bin/attn_trace 4 1024 16 b 100 > gpurun_out/r02al_bwd_trace_cta100.txt 2>&1
./scripts/_bin/attn_trace 4 1024 16 f 200 > gpurun_out/r02al_fwd_trace_cta200.txt 2>&1
cat gpurun_out/r02al_bwd_trace_cta0.txt | head -30
