"""Shared fixtures.  ``-m gpu`` tests need a B200 and the built .so;
everything else runs on the CPU (oracle, host logic, C-ABI exports)."""

import base64
import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "golden.json.gz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU and liblaneutf_b200.so")
    config.addinivalue_line("markers", "slow: long-running sweep")


@pytest.fixture(scope="session")
def golden():
    with gzip.open(GOLDEN_PATH, "rt") as fh:
        g = json.load(fh)
    for key in ("utf8_to_utf16", "utf16_to_utf8"):
        for case in g[key]:
            case["input_bytes"] = base64.b64decode(case["input"])
    return g


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    from paper_2212_05098_b200 import _native

    reason = _native.unavailable_reason()
    if reason is not None:
        if torch.cuda.is_available():
            # a GPU box without the native engine is a failure, not a skip
            pytest.fail(f"native engine unavailable on a GPU box: {reason}")
        pytest.skip(reason)
    return True
