import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def ref():
    import oracle
    return oracle.Reference()


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Restatement()


@pytest.fixture(scope="session")
def default_pairs(ref):
    return ref.generate_pattern(4096, 26, 4.0, 42)


@pytest.fixture(scope="session")
def _session_ctx():
    import paper_1402_2020_b200 as bsm
    return bsm.Context(0)


@pytest.fixture
def ctx(_session_ctx):
    """The session's device context; under BSM_GUARD=1 (guarded device
    buffers, see bsm_debug_check_guards) every test that used it must leave
    all guard bytes intact."""
    yield _session_ctx
    if os.environ.get("BSM_GUARD") == "1":
        damaged, on = _session_ctx.debug_check_guards()
        assert on and damaged == 0, f"{damaged} guard bytes overwritten"


def random_u8(h, w, seed):
    return np.random.default_rng(seed).integers(0, 256, size=(h, w), dtype=np.uint8)
