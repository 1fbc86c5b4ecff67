import json, sys
import numpy as np
sys.path.insert(0, ".")
from oracle import gpt_oracle as O
from paper_2107_06925_b200 import pipesim as P
from paper_2107_06925_b200.gpt import PRESETS, Trainer, synthetic_batch
shape = PRESETS["tiny"]
cfg = P.PipelineConfig(*sys.argv[1].split(",")[:1], *map(int, sys.argv[1].split(",")[1:6])) if len(sys.argv) > 1 else P.PipelineConfig("chimera", 4, 1, 4, 2, 1)
lr = 0.5
tr = Trainer(shape, cfg, lr=lr)
tr.init_params(0)
params = [tr.get_params(s).astype(np.float64) for s in range(cfg.D)]
tok, lab = synthetic_batch(shape, cfg.mini_batch(), 10)
tr.set_batch(tok, lab)
loss = tr.step()
_, ref_loss, g_ref, _ = O.run_iteration(json.loads(tr.schedule_text), O.Shape(**shape.__dict__), params, tok, lab, lr)
print("loss", loss, ref_loss)
for s in range(cfg.D):
    after = tr.get_params(s).astype(np.float64)
    g = (params[s] - after) / lr
    lay, _ = O.stage_layout(O.Shape(**shape.__dict__), cfg.D, s)
    for n, o, r, c, _ in lay:
        a, b = g[o:o + r * c], g_ref[s][o:o + r * c]
        rel = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
        if rel > 0.02:
            print(f"stage {s} {n:24s} rel {rel:.3e} |g| {np.linalg.norm(a):.3e} |ref| {np.linalg.norm(b):.3e}")
    print("stage", s, "total rel", np.linalg.norm(g - g_ref[s]) / np.linalg.norm(g_ref[s]))
