import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box with -m gpu)")


class _Golden(dict):
    @property
    def files(self):
        return list(self.keys())


def load_golden(name: str):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    with np.load(path) as z:  # eager: NpzFile is not thread-safe (ranks run as threads)
        return _Golden({k: z[k] for k in z.files})


@pytest.fixture
def golden():
    return load_golden


@pytest.fixture(scope="session")
def gpu():
    import paper_1908_07038_b200 as sg

    if sg._native.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    sg.set_device(0)
    return sg
