import gzip
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running parity at production size")


def golden_graph(name, tmpdir):
    """Decompress tests/golden/<name>.heops.gz into tmpdir and return its path."""
    src = os.path.join(GOLDEN, f"{name}.heops.gz")
    dst = os.path.join(str(tmpdir), f"{name}.heops")
    if not os.path.exists(dst):
        with gzip.open(src, "rb") as fi, open(dst, "wb") as fo:
            shutil.copyfileobj(fi, fo)
    return dst


@pytest.fixture(scope="session")
def golden_dir(tmp_path_factory):
    return tmp_path_factory.mktemp("golden")
