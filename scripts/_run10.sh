mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpt_gpu.py -m gpu -q --timeout 120 -x -k "backward_pair_fusion or pair_fusion_matches" > gpurun_out/r02k_pairs.log 2>&1
tail -3 gpurun_out/r02k_pairs.log
timeout 120 python scripts/debug_wide.py xl 64 > gpurun_out/r02k_xl.out 2> gpurun_out/r02k_xl.err
echo "xl rc=$?"
timeout 200 python -m pytest tests/test_gpt_wide_gpu.py -m gpu -q --timeout 150 -k xl > gpurun_out/r02k_xltest.log 2>&1
echo "xltest rc=$?"; tail -5 gpurun_out/r02k_xltest.log
timeout 300 python -m pytest tests/test_gpt_wide_gpu.py -m gpu -q --timeout 150 > gpurun_out/r02k_widetest.log 2>&1
echo "wide rc=$?"; tail -5 gpurun_out/r02k_widetest.log
