mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpt_gpu.py -m gpu -q --timeout 120 -x -k "backward_pair_fusion or pair_fusion_matches" > gpurun_out/r02j_pairs.log 2>&1
tail -30 gpurun_out/r02j_pairs.log
CK_TRACE_ISSUE=1 timeout 180 python scripts/debug_wide.py xl 64 > gpurun_out/r02j_xl.out 2> gpurun_out/r02j_xl.err
echo "rc=$?"
tail -5 gpurun_out/r02j_xl.err
head -5 gpurun_out/r02j_xl.out
