mkdir -p gpurun_out
timeout 300 python scripts/debug_wide.py bert 64 > gpurun_out/r02c_debug_bert.txt 2>&1
timeout 300 python scripts/debug_wide.py bert 0.5 > gpurun_out/r02c_debug_bert_lr05.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 tests/test_gemm_gpu.py -k split > gpurun_out/r02c_split.log 2>&1
tail -3 gpurun_out/r02c_split.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_b2.json 2> gpurun_out/r02c_b2.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --B 1 > gpurun_out/r02c_b1.json 2> gpurun_out/r02c_b1.err
tail -c 400 gpurun_out/r02c_b2.json gpurun_out/r02c_b1.json
