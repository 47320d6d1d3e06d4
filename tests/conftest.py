import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size config runs")
    # the oracle and the product libraries are built in-tree; make sure they exist
    if not os.path.exists(os.path.join(ROOT, "oracle", "_build", "liboracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    lib = os.path.join(ROOT, "paper_2206_02200_b200", "_lib")
    if not (os.path.exists(os.path.join(lib, "libgridshift_cuda.so"))
            and os.path.exists(os.path.join(lib, "libgs_gen.so"))):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2206_02200_b200", "csrc")],
                       check=True)


@pytest.fixture(scope="session")
def kats():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_kats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def engine():
    from paper_2206_02200_b200.gridshift import Engine
    e = Engine(0)  # raises on a box without a device: GPU tests never fall back
    yield e
    e.close()
