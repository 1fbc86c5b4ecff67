import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and runs the CUDA path")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        with open(os.path.join(GOLDEN, name)) as fh:
            return fh.read() if name.endswith("_n4.json") else json.load(fh)
    return load


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference library (oracle/_ref); skips where it was not built."""
    from oracle.libs import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (reference not mounted at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def toy_oracle():
    from oracle.libs import ToyLib
    return ToyLib()


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the product library and the C oracle if absent (no-op when up to date)."""
    import subprocess
    lib = os.path.join(ROOT, "paper_2107_06925_b200", "libchimera.so")
    toy = os.path.join(ROOT, "oracle", "_build", "libtoy_oracle.so")
    if not os.path.exists(lib):
        subprocess.check_call(["make", "-s", "-j8", "-C",
                               os.path.join(ROOT, "paper_2107_06925_b200", "csrc")])
    if not os.path.exists(toy):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "all"])
