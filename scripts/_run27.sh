mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -x -q -k attention > gpurun_out/r02ak_attn_tests.log 2>&1; echo "attn tests rc=$?"; tail -3 gpurun_out/r02ak_attn_tests.log
timeout 300 python scripts/bench_attn.py > gpurun_out/r02ak_attn.jsonl 2>&1; cat gpurun_out/r02ak_attn.jsonl
timeout 300 python scripts/bench_attn.py scale > gpurun_out/r02ak_attn_scale.jsonl 2>&1; cat gpurun_out/r02ak_attn_scale.jsonl
timeout 900 python -m pytest tests/test_gpt_gpu.py tests/test_gpt_wide_gpu.py -x -q > gpurun_out/r02ak_gpt_tests.log 2>&1; echo "gpt tests rc=$?"; tail -3 gpurun_out/r02ak_gpt_tests.log
