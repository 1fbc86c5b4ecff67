mkdir -p gpurun_out
timeout 900 python scripts/gemm_split_sweep.py > gpurun_out/r02f_split_sweep.jsonl 2> gpurun_out/r02f_split_sweep.err
CK_GEMM_SPLIT_BF16=0 timeout 600 python scripts/kernel_trace.py --steps 2 --json gpurun_out/r02f_trace_b2_nosplit.json > gpurun_out/r02f_trace_b2_nosplit.txt 2>&1
timeout 600 python scripts/kernel_trace.py --steps 2 --json gpurun_out/r02f_trace_b2.json > gpurun_out/r02f_trace_b2.txt 2>&1
timeout 900 python -m pytest tests/test_gpt_gpu.py tests/test_ops_gpu.py tests/test_gemm_gpu.py -m gpu -q --timeout 600 -x > gpurun_out/r02f_tests.log 2>&1
tail -3 gpurun_out/r02f_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_b2.json 2> gpurun_out/r02f_b2.err
head -30 gpurun_out/r02f_trace_b2_nosplit.txt
