import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def built():
    """Build the engine library and the oracle (test infrastructure) once per session.
    On the GPU box the prebuilt .so files travel with the snapshot; rebuilding is skipped
    when sources are unchanged (and nvcc is present there too)."""
    from paper_2204_07064_b200 import build as B
    if os.environ.get("SC_SKIP_BUILD") != "1":
        B.build()
        B.build_cpp_tests()
        B.build_oracle()
    return True


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def oracle_model(cfg: int, seed: int = 0, **kw):
    """The ORACLE-side twin of configs.build(cfg, seed): identical weights, but the PQMF
    stages take their filters from the independent design (oracle/pqmf_design.py) instead of
    the product's sc_pqmf_filters — so cfg4 / cfg5 parity checks the product's filter design
    too (the two agree to <= 1e-7, test_host.py::test_pqmf_filters_match_independent_design)."""
    from oracle import pqmf_design
    from paper_2204_07064_b200 import configs
    return configs.build(cfg, seed=seed, pqmf_design=pqmf_design.filters, **kw)



def oracle_twin(model):
    """Oracle-side twin of a built flat Model (PQMF weights from the independent design)."""
    from oracle import pqmf_design
    return pqmf_design.twin(model)
