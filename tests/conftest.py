import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built native library")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")


def refsim_or_skip():
    """The reference prefillsim package (baseline/_ref on the GPU box, installed by
    __graft_entry__.build()); skip, with the reason, when this host has no copy."""
    from paper_2602_16603_b200 import refsim

    try:
        return refsim.load()
    except ImportError as e:
        pytest.skip(str(e))


def pytest_sessionfinish(session, exitstatus):
    """PARITY_REPORT=<path>: write every bf16-vs-fp32 parity check of the session (max-abs and
    relative error per config, tests/parity.py) as JSON."""
    path = os.environ.get("PARITY_REPORT")
    if not path:
        return
    try:
        import parity
    except ImportError:
        return
    import json

    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "w") as fh:
        json.dump({"tolerances": {"logits": {"max_abs_frac": parity.LOGIT_ATOL_FRAC,
                                             "rel_l2": parity.LOGIT_REL_TOL},
                                  "kv": {"max_abs_frac": parity.KV_ATOL_FRAC,
                                         "rel_l2": parity.KV_REL_TOL}},
                   "checks": parity.RECORDS}, fh, indent=1)
