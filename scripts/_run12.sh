mkdir -p gpurun_out
for rpw in 1 2 4; do for M in 1264 2528; do CK_LN_BWD_RPW=$rpw timeout 120 python scripts/bench_small_ops.py $M 1280 5120 >> gpurun_out/r02q_small_ops.jsonl 2>/dev/null; done; done
timeout 300 python scripts/bench_attn.py > gpurun_out/r02q_attn.jsonl 2> gpurun_out/r02q_attn.err
timeout 600 python scripts/kernel_trace.py --steps 2 --json gpurun_out/r02q_trace_b2.json > gpurun_out/r02q_trace_b2.txt 2>&1
cat gpurun_out/r02q_small_ops.jsonl | grep ln_
cat gpurun_out/r02q_attn.jsonl
head -25 gpurun_out/r02q_trace_b2.txt
