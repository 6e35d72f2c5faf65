"""The reference-side binding (integration/laneutf_b200_stub.py) and the
reference campaign fixture, on the CPU.

* The stub is importable as a module and binds every C-ABI entry point it
  uses from liblaneutf_b200.so (no GPU needed to load it).
* tests/golden/campaign.npz is exactly what the reference's own campaign
  generator draws (regenerated here from /root/reference when present).
* The oracle agrees with the reference scalar engine on those cases.
"""

import importlib.util
import os
import sys

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"
FIXTURE = os.path.join(ROOT, "tests", "golden", "campaign.npz")


def load_stub():
    path = os.path.join(ROOT, "integration", "laneutf_b200_stub.py")
    spec = importlib.util.spec_from_file_location("laneutf_b200_stub", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def campaign_fixture():
    z = np.load(FIXTURE)
    out = {}
    for direction, tag in (("utf8-to-utf16", "u8"), ("utf16-to-utf8", "u16")):
        data, offs = z[f"{tag}_data"], z[f"{tag}_offsets"]
        out[direction] = [data[offs[i]: offs[i + 1]].tobytes() for i in range(len(offs) - 1)]
    return out


def test_stub_loads_and_binds():
    stub = load_stub()
    for name in ("lu_utf8_to_utf16le", "lu_utf16le_to_utf8", "lu_validate_utf8", "lu_validate_utf16le",
                 "lu_workspace_bytes", "lu_device_supported", "lu_last_error"):
        assert getattr(stub._LIB, name) is not None
    assert stub._LIB.lu_workspace_bytes(stub.OP_UTF8_TO_UTF16LE, 1 << 20) > 0
    import torch

    if not torch.cuda.is_available():
        assert stub.available() is False
    with pytest.raises(ValueError):
        stub.transcode("utf16-to-utf8", b"abc", bytearray(16))  # odd UTF-16 length, before any device work


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")
def test_campaign_fixture_matches_reference_generator():
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from laneutf import difftest
    from make_campaign import SEED, campaign_cases

    fix = campaign_fixture()
    counts = {"utf8-to-utf16": 0, "utf16-to-utf8": 0}
    for direction, data, _m in campaign_cases(difftest, SEED, 300):
        assert data == fix[direction][counts[direction]]
        counts[direction] += 1


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")
def test_oracle_equals_reference_scalar_on_campaign_cases():
    sys.path.insert(0, REF_SRC)
    from laneutf import scalar

    fix = campaign_fixture()
    for data in fix["utf8-to-utf16"][:1500]:
        o, p = scalar.transcode_utf8_to_utf16le(data)
        assert oracle.utf8_to_utf16le(data) == ((o.status.value, o.consumed, o.written), p)
    for data in fix["utf16-to-utf8"][:1500]:
        if len(data) % 2:
            continue
        o, p = scalar.transcode_utf16le_to_utf8(data)
        assert oracle.utf16le_to_utf8(data) == ((o.status.value, o.consumed, o.written), p)
