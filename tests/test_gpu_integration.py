"""The reference-side binding running on the GPU.

integration/laneutf_b200_stub.py -- the ``laneutf/_b200.py`` module of
INTEGRATION.md, loaded as a module; the reference package is not modified
and its ``detect()`` is not patched -- transcodes and validates the
reference's own differential-campaign cases (difftest.py:139-224) and every
result is compared with the oracle:

* the committed fixture (tests/golden/campaign.npz: 2 x 5000 cases the
  reference generator drew, seed 2212) -- always;
* 10^5 live cases per direction drawn by the reference's generator when the
  reference package is installed next to the repo (baseline/_ref travels
  with the snapshot; /root/reference never does).
"""

import os
import sys

import pytest

import oracle

from .test_integration import ROOT, campaign_fixture, load_stub

pytestmark = pytest.mark.gpu

STATUS = {0: "ok", 1: "malformed-input"}


def _check(stub, direction, data):
    if direction == "utf16-to-utf8" and len(data) % 2:
        with pytest.raises(ValueError):
            stub.transcode(direction, data, bytearray(3 * len(data) + 3))
        return
    rec, payload = stub.transcode_to_bytes(direction, data)
    if direction == "utf8-to-utf16":
        ref, ref_payload = oracle.utf8_to_utf16le(data)
        vref = oracle.validate_utf8(data)
    else:
        ref, ref_payload = oracle.utf16le_to_utf8(data)
        vref = oracle.validate_utf16le(data)
    assert (STATUS[rec[0]], rec[1], rec[2]) == ref, (direction, data.hex(), rec, ref)
    assert payload == ref_payload
    v = stub.validate(direction, data)
    assert (STATUS[v[0]], v[1], v[2]) == vref


def test_stub_on_reference_campaign_fixture(cuda_ok):
    stub = load_stub()
    assert stub.available()
    fix = campaign_fixture()
    for direction, cases in fix.items():
        for data in cases:
            _check(stub, direction, data)


@pytest.mark.timeout(1800)
def test_stub_on_live_reference_campaign_1e5(cuda_ok):
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "laneutf")):
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, ref_dir)
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from laneutf import difftest
    from make_campaign import campaign_cases

    stub = load_stub()
    n = 0
    for direction, data, _mutated in campaign_cases(difftest, 2023, 100_000):
        _check(stub, direction, data)
        n += 1
    assert n == 200_000
