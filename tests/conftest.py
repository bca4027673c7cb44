import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _build_native():
    """Build libmemshare.so before any test imports the package (its __init__ loads the .so and
    fails loudly if it is missing). build.py is loaded by path so the package is not imported yet."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_memshare_build",
                                                  os.path.join(ROOT, "paper_2507_21433_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()


def pytest_configure(config):
    _build_native()
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.lib()
    return oracle
