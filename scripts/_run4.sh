mkdir -p gpurun_out
timeout 600 python scripts/gemm_split_sweep.py > gpurun_out/r02d_split_sweep.jsonl 2> gpurun_out/r02d_split_sweep.err
CK_GEMM_SPLIT_BF16=0 timeout 600 python scripts/kernel_trace.py --steps 2 --json gpurun_out/r02d_trace_b2.json > gpurun_out/r02d_trace_b2.txt 2>&1
timeout 900 python -m pytest tests/test_gpt_wide_gpu.py tests/test_reference_suite.py tests/test_toy_gpu.py -m gpu -q --timeout 600 > gpurun_out/r02d_tests.log 2>&1
tail -3 gpurun_out/r02d_tests.log
head -40 gpurun_out/r02d_trace_b2.txt
