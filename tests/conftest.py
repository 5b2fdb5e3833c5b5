import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    if not oracle.ORACLE_SO.exists():
        oracle.build()
    return oracle.load_oracle()


@pytest.fixture(scope="session")
def ref_lib():
    import oracle
    if not oracle.REF_SO.exists():
        if (oracle.REFERENCE_ROOT / "proj" / "include").is_dir():
            oracle.build()
        else:
            pytest.skip("reference driver not built and /root/reference absent")
    return oracle.load_ref()


@pytest.fixture(scope="session")
def gpu_device():
    from paper_2602_18755_b200 import pdsim
    return pdsim.default_device()
