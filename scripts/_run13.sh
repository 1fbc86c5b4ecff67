mkdir -p gpurun_out
timeout 600 python scripts/gemm_wgrad_sweep.py > gpurun_out/r02r_wgrad_sweep.jsonl 2> gpurun_out/r02r_wgrad_sweep.err
cat gpurun_out/r02r_wgrad_sweep.jsonl; tail -3 gpurun_out/r02r_wgrad_sweep.err
