import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

GOLDEN = ROOT / "tests" / "golden"
REF_LIB = ROOT / "oracle" / "_ref" / "libmstab_ref.so"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")


@pytest.fixture(scope="session")
def golden_kat():
    return np.load(GOLDEN / "kat_tridiag.npz")


@pytest.fixture(scope="session")
def golden_seq():
    return np.load(GOLDEN / "seq_small.npz")


@pytest.fixture(scope="session")
def golden_kernels():
    return np.load(GOLDEN / "kernels.npz")


@pytest.fixture(scope="session")
def ref_ctx():
    import paper_1604_06043_b200 as m
    if not REF_LIB.exists():
        pytest.skip("oracle/_ref not built (make ref)")
    return m.Context(m.Lib(REF_LIB))


@pytest.fixture(scope="session")
def gpu_ctx():
    import paper_1604_06043_b200 as m
    return m.Context(m.Lib())
