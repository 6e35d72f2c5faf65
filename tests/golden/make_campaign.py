"""Generate tests/golden/campaign.npz from the reference's own differential
campaign generator (laneutf.difftest, /root/reference/pkg/src/laneutf/
difftest.py:139-224): the cases ``run_campaign(seed=SEED, ...)`` would draw,
exactly, per direction.  Run here (where /root/reference exists); the GPU box
uses the committed fixture.  Expected results are not stored: the tests take
them from the oracle, which tests/test_oracle.py pins to the reference.

    python tests/golden/make_campaign.py [/root/reference/pkg/src]
"""

import os
import sys

import numpy as np

SEED = 2212
CASES = 5000


def campaign_cases(difftest, seed: int, cases_per_direction: int, max_len: int = 4096):
    """Yield (direction, data, was_mutated) in run_campaign's order."""
    from laneutf.corpus import SplitMix64
    from laneutf.engine import DIRECTIONS

    bases = difftest._build_bases(seed)
    for dir_index, direction in enumerate(DIRECTIONS):
        rng = SplitMix64((seed + dir_index) & ((1 << 64) - 1))
        for _ in range(cases_per_direction):
            data, was_mutated = difftest._make_case(rng, bases, direction, max_len)
            yield direction, data, was_mutated


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
    sys.path.insert(0, src)
    from laneutf import difftest

    blobs = {"utf8-to-utf16": [], "utf16-to-utf8": []}
    muts = {"utf8-to-utf16": [], "utf16-to-utf8": []}
    for direction, data, was_mutated in campaign_cases(difftest, SEED, CASES):
        blobs[direction].append(data)
        muts[direction].append(was_mutated)
    arrays = {}
    for key, tag in (("utf8-to-utf16", "u8"), ("utf16-to-utf8", "u16")):
        lens = np.array([len(b) for b in blobs[key]], dtype=np.int64)
        arrays[f"{tag}_data"] = np.frombuffer(b"".join(blobs[key]), dtype=np.uint8)
        arrays[f"{tag}_offsets"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        arrays[f"{tag}_mutated"] = np.array(muts[key], dtype=np.bool_)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "campaign.npz")
    np.savez_compressed(path, seed=np.int64(SEED), **arrays)
    print(path, os.path.getsize(path), {k: v.shape for k, v in arrays.items()})


if __name__ == "__main__":
    main()
