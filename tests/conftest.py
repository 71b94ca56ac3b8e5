import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: full-size parity (BASELINE sizes)")
    # Build every native artefact in-tree once per session (no-op when up to date).
    r = subprocess.run(["make", "-s", "-C", ROOT, "all"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("make failed:\n" + r.stdout[-4000:] + r.stderr[-4000:])


def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not has_gpu():
        pytest.fail("GPU test selected but torch.cuda.is_available() is False")
    import torch

    torch.cuda.init()
    return torch.device("cuda:0")
