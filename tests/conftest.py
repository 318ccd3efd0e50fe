import os
import sys

# tiny complex BLAS calls thrash OpenBLAS threads (10x slower); the oracle is
# vectorised numpy, so pin BLAS to one thread before numpy loads.
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import pytest  # noqa: E402

REFERENCE = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def have_reference():
    return os.path.isdir(REFERENCE)


def rel(a, b):
    import numpy as np
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def pytest_sessionfinish(session, exitstatus):
    """Guard-band builds (tools/canary_run.sh sets PS_CANARY_CHECK): report
    the bytes any kernel wrote past a context allocation during the session."""
    if not os.environ.get("PS_CANARY_CHECK"):
        return
    try:
        from paper_1412_7466_b200 import _lib
        n = _lib.load().ps_canary_check()
    except Exception as e:  # library absent / no GPU
        print(f"\ncanary check unavailable: {e}")
        return
    print(f"\ncanary violations over the test session: {n}")
    if n and n > 0:
        session.exitstatus = 1
