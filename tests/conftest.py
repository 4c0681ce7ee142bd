import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run under gpurun)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def oracle():
    from oracle.py import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.py import Reference
    if not Reference.available():
        pytest.skip("compiled reference (oracle/_ref) not built here")
    return Reference()


@pytest.fixture(scope="session")
def engine():
    from paper_2202_02264_b200.dsmc import Engine
    e = Engine(0)
    yield e
    e.close()


def golden_model(golden, name):
    from tests.cases import CASES, rebuild
    spec = CASES[name]
    pre = f"case_{name}_model_"
    arrays = {k[len(pre):]: v for k, v in golden.items() if k.startswith(pre)}
    return spec, rebuild(spec, arrays)
