mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02bs_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/r02bs_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
