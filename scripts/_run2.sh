mkdir -p gpurun_out
export CUDA_MODULE_LOADING=LAZY
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_b2.json 2> gpurun_out/r02b_b2.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --B 1 > gpurun_out/r02b_b1.json 2> gpurun_out/r02b_b1.err
CK_GEMM_SPLIT_BF16=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_b2_nosplit.json 2> gpurun_out/r02b_b2_nosplit.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r02b_gputests.log 2>&1
tail -3 gpurun_out/r02b_gputests.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 tests/test_gpt_wide_gpu.py tests/test_reference_suite.py tests/test_toy_gpu.py > gpurun_out/r02b_newtests.log 2>&1
tail -3 gpurun_out/r02b_newtests.log
for f in gpurun_out/r02b_b*.json; do echo $f; tail -c 600 $f; done
