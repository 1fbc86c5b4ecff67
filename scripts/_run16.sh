mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -m gpu -q -k "attn or attention" --timeout 300 > gpurun_out/r02u_attn_tests.log 2>&1
tail -3 gpurun_out/r02u_attn_tests.log
timeout 300 python scripts/bench_attn.py > gpurun_out/r02u_attn.jsonl 2>&1
cat gpurun_out/r02u_attn.jsonl
bash scripts/_run15.sh > /dev/null 2>&1
head -12 gpurun_out/r02t_attn_trace_fwd.txt
