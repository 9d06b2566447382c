import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # tests are allowed to use the oracle (checker only)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (full 1024^2 decode against the CPU oracle)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def lbx():
    import paper_2605_19385_b200 as m
    m.lib()
    dbg = os.environ.get("LBX_GEMM_DEBUG")  # "halo_policy,desc_base_mode" (diagnostic runs only)
    if dbg:
        h, d = (int(v) for v in dbg.split(","))
        m.check(m.lib().lbx_op_set_debug(h, d))
    return m
