"""bench.py host helpers on CPU: the workload's FLOP count, the roofline's GEMM shape
list (what one iteration runs, weighted by how often), and that both arms' lines carry
the same `config` object (the driver compares them)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2107_06925_b200.gpt import PRESETS  # noqa: E402


def test_flops_per_seq_matches_survey():
    # GPT-2 1.3B (L64 h1280 s632 V50257) = 5.408 TFLOP per sequence
    assert abs(PRESETS["gpt2-1.3b"].flops_per_seq() / 1e12 - 5.408) < 0.001


def test_roofline_shapes_cover_one_iteration():
    name, cfg, _ = bench.CONFIGS[bench.DEFAULT_CONFIG]
    sh = PRESETS[name]
    shapes = bench.roofline_shapes(sh, cfg)
    M, h, f = cfg["B"] * sh.seq, sh.hidden, sh.ffn
    keys = {s[:5] for s in shapes}
    assert len(keys) == len(shapes)  # merged
    # forward doubling + recompute with fused backward pairs: every stage GEMM on 2M rows
    for (Mm, N, K, a, b) in [(2 * M, 3 * h, h, 0, 0), (2 * M, h, f, 0, 0), (2 * M, h, 3 * h, 0, 1),
                             (3 * h, h, 2 * M, 1, 1), (f, h, 2 * M, 1, 1)]:
        assert (Mm, N, K, a, b) in keys
    w = {s[:5]: s[5] for s in shapes}
    # the forward GEMMs run twice per fused pair (forward + recompute): 0.5 + 0.5
    assert abs(w[(2 * M, 3 * h, h, 0, 0)] - 1.0) < 1e-12
    # unfused backwards: the recompute / dgrad / wgrad shapes move to M rows
    un = {s[:5] for s in bench.roofline_shapes(sh, cfg, bwd_pair_frac=0.0)}
    assert (M, h, 3 * h, 0, 1) in un and (2 * M, h, 3 * h, 0, 1) not in un


def test_both_arms_share_the_config_object():
    name, cfg, work = bench.CONFIGS[bench.DEFAULT_CONFIG]
    bench.SHAPE_NAME, bench.CFG, bench.WORKLOAD = name, cfg, work
    c1 = bench.config_dict(PRESETS[name], 1)
    assert c1["workload"] == work and c1["global_batch"] == cfg["B"] * cfg["N"] * cfg["W"]
    assert c1 == bench.config_dict(PRESETS[name], 1)
    assert "8 logical ranks on 4 GPU(s)" in bench.config_dict(PRESETS[name], 4)["parallelism"]
