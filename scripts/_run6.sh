mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_b2.json 2> gpurun_out/r02g_b2.err
CK_SERIALIZE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_b2_serial.json 2> gpurun_out/r02g_b2_serial.err
CK_SERIALIZE=1 CK_WGRAD_SIDE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_b2_serial_side.json 2> gpurun_out/r02g_b2_serial_side.err
CK_SERIALIZE=1 timeout 600 python scripts/kernel_trace.py --steps 2 --json gpurun_out/r02g_trace_serial.json > gpurun_out/r02g_trace_serial.txt 2>&1
for f in gpurun_out/r02g_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['mfu']['frac_of_sustained'])"; done
head -30 gpurun_out/r02g_trace_serial.txt
