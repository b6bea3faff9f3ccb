import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")


import pytest  # noqa: E402


@pytest.fixture
def engine_options():
    """Set engine test options (xyzb_test_set_option) for one test; all reset
    to 0 (the engine's own choice) afterwards."""
    from paper_1610_05108_b200 import _lib
    used = []

    def set_(**kw):
        for name, value in kw.items():
            if name == "grouping" and isinstance(value, str):
                value = _lib.GROUPING[value]
            _lib.set_test_option(name, int(value))
            used.append(name)

    yield set_
    for name in used:
        _lib.set_test_option(name, 0)
