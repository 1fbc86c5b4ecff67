"""The C-ABI boundary: libchimera.so loads (no GPU needed) and exports every entry
point declared in include/chimera_ck.h; the Python binding table matches the header."""
import os
import re

from paper_2107_06925_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "chimera_ck.h")


def declared():
    text = open(HEADER).read()
    return re.findall(r"CK_API\s+[\w\s\*]+?\b(\w+)\s*\(", text)


def test_every_declared_symbol_is_exported():
    import paper_2107_06925_b200.gpt  # noqa: F401  (registers the ck_gpt_* signatures)
    import paper_2107_06925_b200.kernels  # noqa: F401
    import paper_2107_06925_b200.toy  # noqa: F401
    names = declared()
    assert len(names) >= 40
    L = _lib.lib()
    for n in names:
        assert hasattr(L, n), f"{n} declared in chimera_ck.h but not exported"
    missing = [n for n in names if n not in _lib.SIGNATURES and n != "ck_link_plan"]
    assert not missing, f"no ctypes signature for {missing}"


def test_reference_headers_present():
    inc = os.path.join(os.path.dirname(HEADER), "pipesim")
    for h in ("core.hpp", "rational.hpp", "schedgen.hpp", "analysis.hpp", "dessim.hpp", "perfmodel.hpp",
              "oracle.hpp"):
        assert os.path.exists(os.path.join(inc, h))


def test_status_codes_and_last_error():
    from paper_2107_06925_b200 import pipesim as P
    try:
        P.generate(P.PipelineConfig("chimera", 5, 1, 4))
    except P.InvalidConfigError as e:
        assert e.status == 2 and "even number of stages" in str(e)
    else:
        raise AssertionError("expected InvalidConfigError")


def test_library_does_not_pin_nccl_before_torch():
    # libchimera.so must not drag a second libnccl.so.2 into the process (torch bundles
    # its own): load the library first, then torch, in a fresh interpreter.
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, '.'); from paper_2107_06925_b200 import _lib; _lib.lib(); "
            "import torch; print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_gpt_executor_rejects_pipedream_before_touching_the_device():
    """The GPT executor is synchronous: PipeDream (per-micro-batch updates under weight
    versions, proj/src/oracle.cpp:205-214) is refused with InvalidConfigError (status
    2) at ck_gpt_create, before any device work -- so this runs without a GPU."""
    import pytest
    from paper_2107_06925_b200 import pipesim as P
    from paper_2107_06925_b200.gpt import PRESETS, Trainer
    with pytest.raises(P.InvalidConfigError):
        Trainer(PRESETS["tiny"], P.PipelineConfig("pipedream", 4, 1, 4), lr=0.1)


def test_replay_measured_equals_reference_bubble_on_uniform_tasks():
    """bench.py's `list_schedule_at_measured_task_times`: the reference list-scheduling
    rule replayed with per-task times.  With uniform F = 1, B = 2 and no stalls it must
    reproduce analysis::bubble_ratio exactly (proj/src/analysis.cpp:99-137)."""
    import json
    from fractions import Fraction
    from paper_2107_06925_b200 import pipesim as P
    from paper_2107_06925_b200.gpt import replay_measured
    for cfg in (P.PipelineConfig("chimera", 4, 1, 4), P.PipelineConfig("chimera", 8, 1, 8),
                P.PipelineConfig("chimera", 4, 1, 8, 2, 1, "forward-doubling"), P.PipelineConfig("dapple", 4, 1, 8)):
        text = P.generate_json(cfg, None, -1)
        sched = json.loads(text)
        tasks = [{"rank": w, "kind": t["kind"], "pipeline": t["pipeline_id"], "micro": t["micro_batch"],
                  "stage": t["stage"], "start_ms": 0.0, "end_ms": 1.0 if t["kind"] == "Forward" else 2.0}
                 for w, wl in enumerate(sched["per_worker"]) for t in wl]
        rp = replay_measured({"tasks": tasks}, text)
        want = P.bubble_ratio(text)
        assert abs(rp["per_worker"][0] - float(Fraction(str(want)))) < 1e-12, (cfg, rp, want)
