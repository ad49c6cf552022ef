import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


@pytest.fixture(scope="session")
def golden_kernels():
    import numpy as np

    with np.load(GOLDEN / "kernels.npz") as z:
        data = {k: z[k] for k in z.files}
    shapes = sorted({k.split("/")[0] for k in data})
    return data, shapes


@pytest.fixture(scope="session")
def golden_solves():
    import json

    return json.loads((GOLDEN / "solves.json").read_text())


@pytest.fixture(scope="session")
def golden_precond():
    import json

    return json.loads((GOLDEN / "solves_precond.json").read_text())


@pytest.fixture(scope="session")
def golden_channels():
    import json

    return json.loads((GOLDEN / "solves_channels.json").read_text())


@pytest.fixture(scope="session")
def golden_f32():
    import json

    return json.loads((GOLDEN / "solves_f32.json").read_text())
