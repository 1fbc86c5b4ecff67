"""The reference's OWN test programs, compiled against this repository's drop-in
headers (include/pipesim) and linked to libchimera.so (code written
against the reference recompiles against the drop-in).

* `oracle/_ref/reftests_host`: proj/tests/test_{core,schedgen,analysis,dessim,perfmodel}.cpp
  (79 doctest cases; doctest itself is absent from the image, oracle/doctest_shim stands in);
* `oracle/_ref/reftests_oracle`: proj/tests/test_oracle.cpp -- run_iteration,
  sequential_sgd, check_gradients, PipeDream versioning, missing activations, now
  executed by the GPU ToyModel executor;
* `oracle/_ref/acceptance`: proj/tests/acceptance.cpp, criteria 1-10 (criterion 6 and
  7 run the GPU executor).

The binaries are built by `make -C oracle reftests` (from __graft_entry__.build()) where
/root/reference is mounted and travel to the GPU box as built artefacts."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def _run(name, env=None, timeout=600):
    path = os.path.join(REF, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (reference not mounted at build time)")
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([path], capture_output=True, text=True, timeout=timeout, env=e, cwd=ROOT)


def test_reference_unit_tests_host():
    r = _run("reftests_host")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed | assertions:" in r.stdout and "79 passed" in r.stdout, r.stdout


def test_gpu_entry_without_device_reports_status_3():
    """No sm_100 device (this container): the GPU executor fails loudly with status 3
    and a device message -- never a silent CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2107_06925_b200 import pipesim as P
    from paper_2107_06925_b200 import toy
    from paper_2107_06925_b200._lib import CKError
    cfg = P.PipelineConfig("chimera", 4, 1, 4)
    dims = [4, 4, 5, 3, 3]
    p0 = toy.make_model(dims, 0)
    x, t = toy.make_batch(dims, cfg.mini_batch(), 1)
    with pytest.raises(CKError) as e:
        toy.run_iteration(P.generate_json(cfg, None, -1), dims, p0, x, t, 0.05)
    assert e.value.status == 3 and "cuda" in str(e.value).lower()


@pytest.mark.gpu
def test_reference_unit_tests_oracle_on_gpu():
    r = _run("reftests_oracle")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed | assertions:" in r.stdout, r.stdout


def _criteria(text):
    return [ln for ln in text.splitlines() if ln.startswith("criterion")]


@pytest.mark.gpu
def test_reference_acceptance_on_gpu():
    """Same report as the reference build's own run (proj/test_output.txt, frozen in
    tests/golden/acceptance_reference_output.txt): criteria 2-10 PASS and criterion 1
    FAIL with the identical detail -- the reference itself fails it (GEMS D=2 N=2 is
    fixed at 5/11, outside the closed form's +-0.05).  Every line is byte-identical except
    criterion 7's finite-difference error, which here comes from the GPU fp64 kernels."""
    r = _run("acceptance", env={"PIPESIM_GOLDEN_DIR": os.path.join(ROOT, "tests", "golden")})
    with open(os.path.join(ROOT, "tests", "golden", "acceptance_reference_output.txt")) as fh:
        want = _criteria(fh.read())
    got = _criteria(r.stdout)
    assert len(got) == len(want) == 10, r.stdout + r.stderr
    for g, w in zip(got, want):
        if w.startswith("criterion 7 "):
            assert g.startswith("criterion 7  PASS  finite-difference gradient check"), g
            assert float(g.split("error ")[1].rstrip("]")) <= 1e-10, g
        else:
            assert g == w, (g, w)
    assert "1 criterion(s) failed" in r.stdout
