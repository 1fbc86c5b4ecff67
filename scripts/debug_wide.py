"""Per-tensor gradient norms of one GPU iteration vs the wide fixtures (debug aid)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.make_gpt_wide_fixtures import CASES  # noqa: E402
from paper_2107_06925_b200 import pipesim as P  # noqa: E402
from paper_2107_06925_b200.gpt import GPTShape, Trainer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert"
lr = float(sys.argv[2]) if len(sys.argv) > 2 else 64.0
gold = dict(np.load(os.path.join(ROOT, "tests", "golden", "gpt_wide.npz")))
sh, cf = CASES[name]
tr = Trainer(GPTShape(**sh), P.PipelineConfig(**cf), lr=lr)
tr.init_params(0)
before = {st["stage"]: tr.get_params(st["stage"]).astype(np.float64) for st in tr.layout}
tr.set_batch(gold[f"{name}/tokens"], gold[f"{name}/labels"])
loss = tr.step()
print("loss", loss, "ref", gold[f"{name}/loss"][0])
for st in tr.layout:
    s = st["stage"]
    after = tr.get_params(s).astype(np.float64)
    g = (before[s] - after) / lr
    for t in st["tensors"][:6] + st["tensors"][-3:]:
        key = f"{name}/s{s}/{t['name']}"
        gt = g[t["offset"]:t["offset"] + t["rows"] * t["cols"]]
        b = before[s][t["offset"]:t["offset"] + t["rows"] * t["cols"]]
        print(f"{key:28s} off {t['offset']:10d} {t['rows']}x{t['cols']} mine {np.linalg.norm(gt):.4e} "
              f"ref {float(gold[key + '/norm'][0]):.4e} |w| {np.linalg.norm(b):.4e} max|dw| {np.abs(gt).max():.3e}")
    if s > 1:
        break

from oracle import gpt_oracle as O  # noqa: E402
m = O.Shape(**sh)
ref_params = O.init_params(m, cf["D"], 0)
for st in tr.layout:
    s = st["stage"]
    lay, tot = O.stage_layout(m, cf["D"], s)
    same = [(t["name"], t["offset"], t["rows"], t["cols"]) for t in st["tensors"]] == [(n, o, r, c) for n, o, r, c, _ in lay]
    print("stage", s, "layout equal", same, "numel", st["numel"], tot,
          "max |init diff|", float(np.abs(before[s] - ref_params[s]).max()))
