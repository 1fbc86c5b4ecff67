mkdir -p gpurun_out
T0=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r02w_tests.log 2>&1
echo "tests rc=$? $(( $(date +%s) - T0 ))s"; tail -3 gpurun_out/r02w_tests.log
T0=$(date +%s)
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02w_smoke.log 2>&1
echo "smoke rc=$? $(( $(date +%s) - T0 ))s"; tail -3 gpurun_out/r02w_smoke.log
T0=$(date +%s)
timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err
echo "bench rc=$? $(( $(date +%s) - T0 ))s"
T0=$(date +%s)
timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02w_ref.json 2> gpurun_out/r02w_ref.err
echo "ref rc=$? $(( $(date +%s) - T0 ))s"
tail -c 3000 gpurun_out/r02w_bench.json; echo; cat gpurun_out/r02w_ref.json
