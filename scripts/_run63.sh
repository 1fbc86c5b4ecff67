# final-build ncu launch list of one graph-replayed step of the bench workload
mkdir -p gpurun_out
timeout 600 python scripts/step_profile.py --steps 1 > gpurun_out/r02bq_step.json 2>&1 || exit 1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02bq_launches.csv python scripts/step_profile.py --steps 1 > gpurun_out/r02bq_ncu_launch.log 2>&1
echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/r02bq_launches.csv > gpurun_out/r02bq_launch_summary.txt
head -20 gpurun_out/r02bq_launch_summary.txt
