mkdir -p gpurun_out
timeout 300 python scripts/attn_once.py > gpurun_out/r02bn_once.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_attn_.*_tc" -c 2 -o gpurun_out/r02bn_attn python scripts/attn_once.py > gpurun_out/r02bn_ncu.log 2>&1
echo "ncu rc=$?"
