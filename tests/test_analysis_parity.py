"""Live-reference parity of the schedule metrics layer (SURVEY.md §8(a) a23-a28,
§8(f)-3): analysis::validate_dependencies (incl. malformed schedules), bubble per
worker, steady-state idle, memory_profile, perfmodel::free_regions / critical_path /
predict_T / plan and dessim::simulate, each compared EXACTLY (parsed JSON doubles)
against the unmodified reference library built in oracle/_ref.

These tests are the gate for the independent rewrites of schedgen / analysis /
dessim / perfmodel (VERDICT r01 copy remediation)."""
import json
import random

import pytest

from paper_2107_06925_b200 import pipesim as P

SCALINGS = ["direct", "forward-doubling", "backward-halving"]


def _lattice(n, seed):
    rng = random.Random(seed)
    out = []
    while len(out) < n:
        scheme = rng.choice(["chimera"] * 5 + ["gpipe", "dapple", "gems", "pipedream", "pipedream-2bw"])
        D = rng.choice([2, 4, 6, 8])
        f = rng.choice([x for x in range(1, D // 2 + 1) if (D // 2) % x == 0]) if scheme == "chimera" else 1
        N = rng.choice([1, 2, D - 1, D, D + 1, 2 * D, 3 * D, 4 * D])
        sc = rng.choice(SCALINGS) if scheme == "chimera" else "direct"
        B = rng.choice([1, 2, 4])
        prof = P.CostProfile(backward_ratio=rng.choice([1.0, 1.5, 2.0, 3.0, 4.0 / 3.0]),
                             F_t=rng.choice([1.0, 0.37, 2.5]),
                             alpha=rng.choice([0.0, 0.013, 0.2]), beta=rng.choice([0.0, 0.0007, 0.01]),
                             L_grad=rng.choice([0.0, 64.0, 123.0]), L_act=rng.choice([0.0, 3.5]),
                             M_a=rng.choice([1.0, 2.0]), M_a_ckpt=0.5, M_theta=rng.choice([1.0, 3.0]),
                             embed_surcharge=rng.choice([False, True]))
        out.append((P.PipelineConfig(scheme, D, rng.choice([1, 2]), N, B, f, sc), prof))
    return out


def _mutations(sched: dict, rng):
    """Malformed variants of a valid schedule: each breaks one invariant that
    validate_dependencies checks (proj/src/analysis.cpp:40-95)."""
    pw = sched["per_worker"]
    out = []
    w = rng.randrange(len(pw))
    if len(pw[w]) >= 2:  # swap two neighbours: may reorder stages or create a cycle
        i = rng.randrange(len(pw[w]) - 1)
        m = json.loads(json.dumps(sched))
        m["per_worker"][w][i], m["per_worker"][w][i + 1] = m["per_worker"][w][i + 1], m["per_worker"][w][i]
        out.append(m)
        m = json.loads(json.dumps(sched))  # reverse a worker: cycles / out-of-order stages
        m["per_worker"][w].reverse()
        out.append(m)
    m = json.loads(json.dumps(sched))  # duplicate a task
    m["per_worker"][w].append(dict(m["per_worker"][w][0]))
    out.append(m)
    m = json.loads(json.dumps(sched))  # duplicate a backward: stage order + duplicate
    m["per_worker"][w].append(dict(m["per_worker"][w][-1]))
    out.append(m)
    fw = [(ww, i) for ww, lst in enumerate(pw) for i, t in enumerate(lst) if t["kind"] == "Forward"]
    ww, i = rng.choice(fw)  # drop a forward: orphan backward
    m = json.loads(json.dumps(sched))
    del m["per_worker"][ww][i]
    out.append(m)
    return out


def test_live_analysis_report_lattice(ref):
    rng = random.Random(7)
    n = 0
    for cfg, prof in _lattice(160, 99):
        try:
            text = ref.generate(cfg.to_json(), prof.to_json(), -1)
        except RuntimeError:
            continue
        assert P.generate_json(cfg, prof, -1) == text
        want = ref.analysis_report(text, prof.to_json())
        got = P.analysis_report(text, prof)
        assert got == want, (cfg, prof)
        for m in _mutations(json.loads(text), rng):
            mt = json.dumps(m)
            assert P.analysis_report(mt, prof) == ref.analysis_report(mt, prof.to_json()), (cfg, m)
        n += 1
    assert n > 100


def test_live_predict_T_and_simulate(ref):
    n = 0
    for cfg, prof in _lattice(120, 5):
        try:
            text = ref.generate(cfg.to_json(), prof.to_json(), -1)
        except RuntimeError:
            continue
        assert P.predict_T(cfg, prof) == ref.predict_T(cfg.to_json(), prof.to_json()), (cfg, prof)
        for pol, name in enumerate(P.POLICIES):
            for zc in (False, True):
                want = ref.simulate(text, prof.to_json(), pol, zc)
                got = P.simulate(text, prof, name, zero_comm=zc)
                assert json.dumps(got["timed"]) == json.dumps(want["timed"])
                assert got["allreduce_events"] == want["allreduce_events"]
                assert got["per_worker_idle"] == want["per_worker_idle"]
                for k in ("makespan", "compute_makespan", "allreduce_exposed"):
                    assert got[k] == want[k], (cfg, name, k)
        n += 1
    assert n > 80


@pytest.mark.parametrize("scheme", ["chimera", "dapple", "gpipe", "gems"])
def test_live_plan(ref, scheme):
    rng = random.Random(11)
    for _ in range(6):
        prof = P.CostProfile(backward_ratio=rng.choice([2.0, 1.5]), F_t=rng.choice([1.0, 0.75]),
                             alpha=rng.choice([0.0, 0.01]), beta=rng.choice([0.0, 1e-3]),
                             L_grad=rng.choice([0.0, 100.0]), L_act=rng.choice([0.0, 4.0]),
                             M_a=rng.choice([1.0, 4.0]), M_a_ckpt=1.0, M_theta=2.0,
                             mem_capacity=rng.choice([1e18, 60.0, 30.0]))
        for Pn, Bh in ((2, 16), (4, 32), (8, 64), (6, 24)):
            try:
                want = ref.plan(Pn, Bh, prof.to_json(), scheme)
            except RuntimeError as e:
                with pytest.raises(P.CKError):
                    P.plan(Pn, Bh, prof, scheme)
                assert "no (W, D, B)" in str(e) or "plan requires" in str(e)
                continue
            assert P.plan(Pn, Bh, prof, scheme) == want, (Pn, Bh, prof)
