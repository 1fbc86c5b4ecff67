"""Pins the numpy transformer oracle (oracle/gpt_oracle.py) -- CPU only.

The reference has no transformer, so the oracle is pinned by the reference's own
properties: pipelined Chimera == sequential mini-batch SGD (<= 1e-10 in fp64,
proj/tests/test_oracle.cpp:92-109) and central finite differences
(proj/src/oracle.cpp:358-410, <= 1e-5)."""
import json

import numpy as np

from oracle import gpt_oracle as O
from paper_2107_06925_b200 import pipesim as P

MICRO = O.Shape(n_layer=4, hidden=128, heads=2, ffn=256, seq=16, vocab=50, vocab_padded=64, causal=True)


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_layout_matches_product_convention():
    # the product (C++) and the oracle pack stage tensors identically
    from paper_2107_06925_b200.gpt import PRESETS
    s = PRESETS["tiny"]
    for D in (2, 4):
        for st in range(D):
            lay, tot = O.stage_layout(O.Shape(**s.__dict__), D, st)
            assert tot % 64 == 0 and lay[0][1] == 0


def test_pipelined_equals_sequential():
    for cfg in [P.PipelineConfig("chimera", 4, 2, 4, 2, 1), P.PipelineConfig("chimera", 4, 1, 8, 1, 2),
                P.PipelineConfig("chimera", 2, 1, 4, 2, 1, "forward-doubling"),
                P.PipelineConfig("gpipe", 4, 1, 4, 2)]:
        sched = json.loads(P.generate_json(cfg, None, -1))
        params = O.init_params(MICRO, cfg.D, 3)
        n = cfg.mini_batch()
        tok, lab = O.synthetic_tokens(MICRO, n, 5)
        new, loss, g, peak = O.run_iteration(sched, MICRO, params, tok, lab, 0.1)
        seq_new, seq_loss, seq_g = O.sequential_sgd(MICRO, cfg.D, params, tok, lab, 0.1, n)
        assert abs(loss - seq_loss) <= 1e-10 * abs(seq_loss)
        for s in range(cfg.D):
            assert _rel(g[s], seq_g[s]) <= 1e-10
        assert peak == P.memory_profile(json.dumps(sched))["act_counts"]


def test_finite_differences():
    m = O.Shape(n_layer=2, hidden=128, heads=2, ffn=128, seq=8, vocab=20, vocab_padded=32, causal=True)
    D = 2
    params = O.init_params(m, D, 1)
    params = [p * 5 for p in params]  # larger weights -> non-trivial curvature
    for s in range(D):
        lay, _ = O.stage_layout(m, D, s)
        for n, o, r, c, init in lay:
            if init == "one":
                params[s][o:o + r * c] = 1.0
    tok, lab = O.synthetic_tokens(m, 3, 2)
    _, loss0, g = O.sequential_sgd(m, D, params, tok, lab, 0.0, 3)
    rng = np.random.default_rng(0)
    worst = 0.0
    for s in range(D):
        lay, tot = O.stage_layout(m, D, s)
        for n, o, r, c, _ in lay:
            for idx in rng.integers(o, o + r * c, size=3):
                eps = 1e-5
                pp = [p.copy() for p in params]
                pp[s][idx] += eps
                _, lp, _ = O.sequential_sgd(m, D, pp, tok, lab, 0.0, 3)
                pp[s][idx] -= 2 * eps
                _, lm, _ = O.sequential_sgd(m, D, pp, tok, lab, 0.0, 3)
                fd = (lp - lm) / (2 * eps)
                worst = max(worst, abs(fd - g[s][idx]) / max(1.0, abs(fd), abs(g[s][idx])))
    assert worst <= 1e-5


def test_balanced_partition_prefers_short_head_stage():
    from paper_2107_06925_b200.gpt import PRESETS, balanced_partition
    part = balanced_partition(PRESETS["gpt2-medium"], P.PipelineConfig("chimera", 4, 2, 4, 4, 1))
    assert sum(part) == 24 and part[-1] < part[1]
    m = O.Shape(n_layer=4, hidden=128, heads=2, ffn=256, seq=16, vocab=50, vocab_padded=64, causal=True,
                stage_layers=(2, 1, 1, 0 + 0) if False else (1, 1, 1, 1))
    assert O.stage_layout(m, 4, 3)[0][-1][0] == "lm_head"


def test_balanced_partition_measured_head_cost():
    """The LM head counted at its measured cost (gpt.HEAD_EFFICIENCY) moves a layer to the
    head stage on GPT-2 medium D=4 (measured bubble 0.252 vs the reference's
    0.253); counted at its FLOP ratio the old (7, 7, 7, 3) split comes back."""
    from paper_2107_06925_b200.gpt import HEAD_EFFICIENCY, PRESETS, balanced_partition
    cfg = P.PipelineConfig("chimera", 4, 1, 4, 4, 1)
    assert 0.5 < HEAD_EFFICIENCY < 1.0
    assert balanced_partition(PRESETS["gpt2-medium"], cfg) == (7, 6, 7, 4)
    assert balanced_partition(PRESETS["gpt2-medium"], cfg, 1.0) == (7, 7, 7, 3)
    for name in ("gpt2-medium", "gpt2-1.3b", "bert48"):
        sh = PRESETS[name]
        for D in (4, 8):
            part = balanced_partition(sh, P.PipelineConfig("chimera", D, 1, 2 * D, 1, 1))
            assert sum(part) == sh.n_layer and min(part) >= 1
