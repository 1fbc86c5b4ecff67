mkdir -p gpurun_out
for v in "X=1" "CK_LN_BWD_SKIP_ATOMICS=1" "CK_LN_BWD_RPW=2" "CK_LN_BWD_RPW=4" "CK_LN_BWD_RPW=4 CK_LN_BWD_SKIP_ATOMICS=1"; do
  echo "== $v"; env $v timeout 120 python scripts/bench_small_ops.py 2528 1280 5120 2>&1 | grep ln_
  env $v timeout 120 python scripts/bench_small_ops.py 1264 1280 5120 2>&1 | grep ln_bwd
done
