timeout 300 python scripts/bench_attn.py breakdown 2>/dev/null
