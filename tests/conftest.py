import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden_cases(prefix=None):
    """Names of the golden fixtures: run_pipeline cases (prefix None), or the
    ``pb_`` (run_pixel_baseline) / ``seam_`` / ``metrics_`` ones."""
    import glob

    names = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))
    if prefix is None:
        return [n for n in names if not n.startswith(("seam_", "pb_", "metrics_", "files_"))]
    return [n for n in names if n.startswith(prefix)]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
