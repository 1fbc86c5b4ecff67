mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -x -q -k attention 2>&1 | tail -2
timeout 300 python scripts/bench_attn.py 2>&1
timeout 300 python scripts/bench_attn.py breakdown 2>/dev/null
