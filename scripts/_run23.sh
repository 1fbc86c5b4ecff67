mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -m gpu -q -k "attn or attention" --timeout 300 > gpurun_out/r02ab_attn_tests.log 2>&1
tail -2 gpurun_out/r02ab_attn_tests.log
timeout 300 python scripts/bench_attn.py > gpurun_out/r02ab_attn.jsonl 2>&1
cat gpurun_out/r02ab_attn.jsonl
