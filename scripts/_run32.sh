mkdir -p gpurun_out
for M in 1264 2528 4096; do timeout 120 python scripts/bench_small_ops.py $M 1280 5120 2>&1 | grep "op\": \"ln_"; done
timeout 120 python scripts/bench_small_ops.py 4096 1024 4096 2>&1 | grep "op\": \"ln_"
