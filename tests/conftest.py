import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running parity case")
    # the CPU-side shared libraries are cheap to build; make sure they exist
    need = [os.path.join(ROOT, "oracle", "liboracle.so"), os.path.join(ROOT, "gen", "libgen.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-C", ROOT, "oracle", "gen"], check=True)
