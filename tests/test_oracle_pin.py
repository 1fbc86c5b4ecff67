"""Pins the C restatement of the ToyModel oracle (oracle/toy_oracle.c) before any GPU
result is compared with it: against the golden fixtures produced by the unmodified
reference (tests/golden/toy_oracle.json; SURVEY.md Appendix D.3 known answers) and,
where it is built, against the live reference library."""
import json

import numpy as np
import pytest

from oracle.libs import tasks_of  # noqa: F401  (layout helper shared with the GPU tests)
from paper_2107_06925_b200 import pipesim as P


def test_generators_bit_exact(golden, toy_oracle):
    g = golden("toy_oracle.json")["generators"]
    assert np.array_equal(toy_oracle.make_model(g["dims"], 42), np.array(g["model42"]))
    x, t = toy_oracle.make_batch(g["dims"], 16, 100)
    assert np.array_equal(x, np.array(g["batch100_inputs"]))
    assert np.array_equal(t, np.array(g["batch100_targets"]))
    # SURVEY.md D.3
    assert g["model42"][0] == 0.12757776647726948
    assert g["batch100_inputs"][0] == 0.36561232062294402


def test_run_iteration_matches_reference_fixtures(golden, toy_oracle):
    for case in golden("toy_oracle.json")["cases"]:
        c, dims = case["config"], case["dims"]
        sched = json.loads(P.generate_json(P.PipelineConfig(**c), None, -1))
        params = toy_oracle.make_model(dims, case["model_seed"])
        batch = c["B"] * c["N"] * c["W"]
        for it, seed in enumerate(case["batch_seeds"]):
            x, t = toy_oracle.make_batch(dims, batch, seed)
            params, peaks = toy_oracle.run_iteration(sched, dims, params, x, t, case["lr"])
            # identical arithmetic order -> bit-identical to the reference
            assert np.array_equal(params, np.array(case["params_after"][it])), (c, it)
        assert peaks == case["peak_stash"]
        seq = np.array(case["sequential_after3"])
        assert toy_oracle.max_relative_diff(dims, params, seq) <= 1e-6


def test_known_answer_d3(golden):
    case = golden("toy_oracle.json")["cases"][0]
    assert case["config"] == {"scheme": "chimera", "D": 4, "W": 2, "N": 4, "B": 2, "f": 1,
                              "scaling": "direct", "recompute": False}
    final = case["params_after"][-1]
    assert final[0] == 0.12758666599534998 and final[1] == 0.069536694131678553


def test_sequential_sgd_matches_reference(ref, toy_oracle):
    dims = [4, 5, 4, 3]
    p = ref.make_model(dims, 7)
    x, t = ref.make_batch(dims, 12, 3)
    assert np.array_equal(ref.sequential_sgd(dims, p, x, t, 12, 0.1),
                          toy_oracle.sequential_sgd(dims, p, x, t, 12, 0.1))


def test_list_schedule_matches_reference(ref, toy_oracle):
    for cfg in [P.PipelineConfig("chimera", 8, 1, 32, 1, 1, "forward-doubling"),
                P.PipelineConfig("chimera", 8, 1, 16, 1, 2)]:
        text = P.generate_json(cfg, None, -1)
        sim = ref.simulate(text, P.CostProfile().to_json(), 0, zero_comm=True)
        st, en, mk = toy_oracle.list_schedule(json.loads(text), 1.0, 2.0)
        want = [sp["start"] for wl in sim["timed"]["timing"] for sp in wl]
        assert st.tolist() == want and mk == sim["makespan"]
