"""TEST INFRASTRUCTURE ONLY -- freeze numpy fp64 oracle results (oracle/gpt_oracle.py)
for the GPT stage executor at the BENCHMARKED widths, so the GPU box (which has no
time for fp64 numpy at these sizes) checks one Chimera iteration against them.

    python -m oracle.make_gpt_wide_fixtures        # ~2-4 min on 8 cores

Cases (reduced depth, full width -- VERDICT r01 "next round" item 1):
  * medium:  h=1024, 16 heads, s=1024, V=50257 (50304 padded), 4 layers, Chimera D=4
             N=4 W=2 B=1 (configs[1] width);
  * xl:      h=1280, 20 heads, s=632, V=50257, 6 layers split (2,1,2,1), Chimera D=4
             N=8 forward-doubling + recompute, B=1 (configs[3] width; the executor
             fuses each virtual micro-batch's two forwards into one 1264-row pass);
  * bert:    h=1024, 16 heads, s=128, V=30522 (30592), bidirectional, 8 layers,
             Chimera D=8 N=8 B=1 (configs[2] width).
For every case: tokens/labels, the mean loss, and per stage and per tensor the
gradient's L2 norm plus its values at a fixed index sample (every element of vectors
<= 8192 long; 2048 deterministic positions of matrices -- for the token embedding,
positions inside rows of tokens that occur).  Written to tests/golden/gpt_wide.npz.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import gpt_oracle as O  # noqa: E402

CASES = {
    "medium": (dict(n_layer=4, hidden=1024, heads=16, ffn=4096, seq=1024, vocab=50257, vocab_padded=50304,
                    causal=True, stage_layers=(1, 1, 1, 1)),
               dict(scheme="chimera", D=4, W=2, N=4, B=1, f=1, scaling="direct", recompute=False)),
    "xl": (dict(n_layer=6, hidden=1280, heads=20, ffn=5120, seq=632, vocab=50257, vocab_padded=50304,
                causal=True, stage_layers=(2, 1, 2, 1)),
           dict(scheme="chimera", D=4, W=1, N=8, B=1, f=1, scaling="forward-doubling", recompute=False)),
    "bert": (dict(n_layer=8, hidden=1024, heads=16, ffn=4096, seq=128, vocab=30522, vocab_padded=30592,
                  causal=False, stage_layers=()),
             dict(scheme="chimera", D=8, W=1, N=8, B=1, f=1, scaling="direct", recompute=False)),
}
SEED_PARAMS, SEED_TOKENS, LR = 0, 5, 64.0


def sample_index(name, rows, cols, tokens):
    n = rows * cols
    if n <= 8192:
        return np.arange(n, dtype=np.int64)
    k = np.arange(2048, dtype=np.int64)
    if name == "wte":
        used = np.unique(tokens)
        r = used[(k * 7919) % len(used)]
        return np.unique(r * cols + (k * 104729) % cols)
    return np.unique((k * 2654435761) % n)


def main(names=None):
    from paper_2107_06925_b200 import pipesim as P
    out = {}
    for name, (sh, cf) in CASES.items():
        if names and name not in names:
            continue
        t0 = time.time()
        m = O.Shape(**sh)
        cfg = P.PipelineConfig(**cf)
        text = P.generate_json(cfg, None, -1)
        sched = json.loads(text)
        D = cfg.D
        # the product's fp32 master weights are these values rounded to fp32
        params = [p.astype(np.float32).astype(np.float64) for p in O.init_params(m, D, SEED_PARAMS)]
        tok, lab = O.synthetic_tokens(m, cfg.mini_batch(), SEED_TOKENS)
        _, loss, g, peak = O.run_iteration(sched, m, params, tok, lab, LR)
        out[f"{name}/tokens"] = tok
        out[f"{name}/labels"] = lab
        out[f"{name}/loss"] = np.array([loss])
        out[f"{name}/peak"] = np.array(peak)
        for s in range(D):
            layout, total = O.stage_layout(m, D, s)
            for tname, off, rows, cols, _ in layout:
                gt = g[s][off:off + rows * cols]
                idx = sample_index(tname, rows, cols, tok)
                key = f"{name}/s{s}/{tname}"
                out[key + "/norm"] = np.array([np.linalg.norm(gt)])
                out[key + "/idx"] = idx
                out[key + "/val"] = gt[idx]
        print(f"{name}: loss {loss:.6f}  peak {peak}  {time.time() - t0:.1f} s", flush=True)
    path = os.path.join(ROOT, "tests", "golden", "gpt_wide.npz")
    if names and os.path.exists(path):
        old = dict(np.load(path))
        old.update(out)
        out = old
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
