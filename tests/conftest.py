import os
import sys

# The golden fixtures were produced with a single-threaded OpenBLAS
# (tests/golden/make_golden.py); a threaded ddot splits the sum differently,
# so the oracle's bitwise pins only hold with one BLAS thread.
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[_v] = "1"

import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

threadpool_limits(1)
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
CASES = ["pack2d", "pack3d", "rand3d", "wrap2", "channel16", "disks2d",
         "spheres3d", "exhaust"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libvoxschur.so")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(params=CASES)
def golden(request):
    return request.param, load_golden(request.param)
