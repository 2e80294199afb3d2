import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / round-end GPU tier)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")
    # temporary files (tmp_path) stay inside the repository
    if not config.option.basetemp:
        config.option.basetemp = str(Path(__file__).resolve().parent.parent / ".pytest_tmp")


@pytest.fixture(scope="session")
def ref_lib():
    """The reference core build (oracle/_ref); built here if the sources exist."""
    from oracle import ref
    if not ref.build_if_possible():
        pytest.skip("reference build oracle/_ref unavailable (no /root/reference and not prebuilt)")
    return ref


@pytest.fixture(scope="session")
def ctx():
    from paper_1602_03207_b200 import ect
    c = ect.Context(int(os.environ.get("ECT_DEVICE", "0")))
    yield c
    c.close()
