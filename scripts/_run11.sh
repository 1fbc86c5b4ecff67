mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > gpurun_out/r02l_tests.log 2>&1
echo "rc=$?"
tail -15 gpurun_out/r02l_tests.log
