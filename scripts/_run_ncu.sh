# ncu evidence for the bench line: (1) launch list of ONE graph-replayed step of the
# default workload (gpu__time_duration.sum, --clock-control none); (2) --set full of the
# roofline GEMM shapes (DRAM traffic per launch, tensor-pipe activity).  Each command is
# first run without ncu.
mkdir -p gpurun_out
timeout 600 python scripts/step_profile.py --steps 1 > gpurun_out/r02n_step.json 2>&1 || exit 1
timeout 2400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02n_launches.csv python scripts/step_profile.py --steps 1 > gpurun_out/r02n_ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/r02n_launches.csv > gpurun_out/r02n_launch_summary.txt
timeout 300 python scripts/roofline_shapes.py > gpurun_out/r02n_shapes.log 2>&1 || exit 1
timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_gemm|k_splitk" \
  -o gpurun_out/r02n_gemm_roofline python scripts/roofline_shapes.py > gpurun_out/r02n_ncu_full.log 2>&1
python scripts/ncu_gemm_roofline.py gpurun_out/r02n_gemm_roofline.ncu-rep gpurun_out/r02n_gemm_roofline.json --config gpt2-1.3b --B 2
head -30 gpurun_out/r02n_launch_summary.txt
