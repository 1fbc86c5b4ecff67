"""Multi-process parity: the tiny GPT under Chimera D=4 W=2 on G processes (one GPU
each) must produce the same loss and weights as the single-process run.
MP_OPT=adamw: both runs use AdamW; MP_OPT=zero: the multi-process run shards the AdamW
moments over each stage's holders (ZeRO-1: reduce-scatter, shard update, all-gather)
while the single-process reference keeps them whole -- same mathematics."""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, ".")
from paper_2107_06925_b200 import pipesim as P
from paper_2107_06925_b200.gpt import PRESETS, Trainer, synthetic_batch

dist.init_process_group("gloo")
world, rank = dist.get_world_size(), dist.get_rank()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) // int(os.environ.get("CK_PROCS_PER_GPU", "1")))
shape = PRESETS["tiny"]
# MP_CFG=fd: forward doubling + recompute (D=4 W=1 N=8), else Chimera D=4 W=2 N=4 direct
cfg = (P.PipelineConfig("chimera", 4, 1, 8, 1, 1, "forward-doubling") if os.environ.get("MP_CFG") == "fd"
       else P.PipelineConfig("chimera", 4, 2, 4, 2, 1))
per = cfg.W * cfg.D // world
LR = 0.5 if os.environ.get("MP_OPT", "sgd") == "sgd" else 1e-3
tr = Trainer(shape, cfg, lr=LR, first_rank=rank * per, n_ranks=per)
tr.connect()
OPT = os.environ.get("MP_OPT", "sgd")
if OPT != "sgd":
    tr.set_optimizer("adamw", 0.9, 0.99, 1e-4, 0.01, zero=OPT == "zero")
tr.init_params(0)
losses = []
for it in range(3):
    tok, lab = synthetic_batch(shape, cfg.mini_batch(), 10 + it)
    tr.set_batch(tok, lab)
    l = torch.tensor([tr.step()])
    dist.all_reduce(l)
    losses.append(float(l))
params = {s: tr.get_params(s) for s in tr.stages}
out = [None] * world
dist.all_gather_object(out, params)
if rank == 0:
    merged = {}
    for d in out:
        for s, v in d.items():
            if s in merged:
                assert np.array_equal(merged[s], v), f"stage {s} copies differ across processes"
            merged[s] = v
    ref = Trainer(shape, cfg, lr=LR)
    if OPT != "sgd":
        ref.set_optimizer("adamw", 0.9, 0.99, 1e-4, 0.01, zero=False)
    ref.init_params(0)
    rl = []
    for it in range(3):
        tok, lab = synthetic_batch(shape, cfg.mini_batch(), 10 + it)
        ref.set_batch(tok, lab)
        rl.append(ref.step())
    md = max(float(np.abs(merged[s] - ref.get_params(s)).max()) for s in range(cfg.D))
    print(json.dumps({"world": world, "cfg": os.environ.get("MP_CFG", "direct"), "opt": OPT, "losses": losses,
                      "ref_losses": rl,
                      "max_abs_param_diff": md}))
    assert md < 1e-3 and all(abs(a - b) <= 1e-4 * abs(b) for a, b in zip(losses, rl)), "multi-process != single"
dist.barrier()
tr.close()
