mkdir -p gpurun_out/timelines
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CK_TIMELINE=gpurun_out/timelines/r02_d4n8fd timeout 900 $TR --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --config gpt2-medium-d4-n8fd --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02m_d4n8fd_n4.json 2> gpurun_out/r02m_d4n8fd_n4.err
for o in sgd adamw zero; do MP_OPT=$o timeout 300 $TR --nproc-per-node 4 --master-port 2953$((RANDOM%9)) scripts/mp_check.py >> gpurun_out/r02m_mp_check.jsonl 2>> gpurun_out/r02m_mp_check.err; done
MP_CFG=fd timeout 300 $TR --nproc-per-node 4 --master-port 29541 scripts/mp_check.py >> gpurun_out/r02m_mp_check.jsonl 2>> gpurun_out/r02m_mp_check.err
cat gpurun_out/r02m_mp_check.jsonl
tail -c 1200 gpurun_out/r02m_d4n8fd_n4.json
