"""Generate the golden parity fixtures from the reference implementation.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``laneutf`` (pure Python) and its own test
vectors, runs the reference scalar oracle (pkg/src/laneutf/scalar.py) on
them and on seeded random/mutated inputs, and writes ``golden.json.gz`` next to
this file.  The fixtures pin the C oracle (oracle/) and, through it, the
CUDA engine.  Nothing here runs on the GPU box.

Sources of the vectors (imported, not retyped):
  * BOUNDARY_ROWS, SAMPLE_UTF8/SAMPLE_WORDS, UTF8_ERROR_CASES,
    UTF16_ERROR_CASES  -- pkg/tests/test_scalar.py:24-36, 84-121
  * SplitMix64 stream -- pkg/src/laneutf/corpus.py:65-82
    (known answers at pkg/tests/test_corpus.py:23-27)
  * corpus.generate / corpus.mutate -- pkg/src/laneutf/corpus.py:152-285
"""

from __future__ import annotations

import base64
import gzip
import hashlib
import importlib
import importlib.util
import json
import os
import random
import sys

REF_PKG = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    sys.path.insert(0, os.path.join(REF_PKG, "src"))
    import laneutf  # noqa: F401
    from laneutf import corpus, scalar

    spec = importlib.util.spec_from_file_location(
        "laneutf_reftests",
        os.path.join(REF_PKG, "tests", "__init__.py"),
        submodule_search_locations=[os.path.join(REF_PKG, "tests")],
    )
    pkg = importlib.util.module_from_spec(spec)
    sys.modules["laneutf_reftests"] = pkg
    spec.loader.exec_module(pkg)
    ref_tests = importlib.import_module("laneutf_reftests.test_scalar")
    return scalar, corpus, ref_tests


def b64(data: bytes) -> str:
    return base64.b64encode(data).decode("ascii")


def payload_field(payload: bytes):
    """Small payloads verbatim; large ones as sha256 (keeps the fixture small)."""
    if len(payload) <= 1024:
        return b64(payload)
    return "sha256:" + hashlib.sha256(payload).hexdigest()


def outcome_tuple(o) -> list:
    return [o.status.value, o.consumed, o.written]


def main() -> None:
    scalar, corpus, T = _import_reference()
    words_to_bytes = T.words_to_bytes

    cases_u8 = []  # (name, input bytes)
    cases_u16 = []

    for cp, utf8_hex, words in T.BOUNDARY_ROWS:
        cases_u8.append((f"boundary-{cp:04X}", bytes.fromhex(utf8_hex)))
        cases_u16.append((f"boundary-{cp:04X}", words_to_bytes(words)))
    cases_u8.append(("sample", T.SAMPLE_UTF8))
    cases_u16.append(("sample", words_to_bytes(T.SAMPLE_WORDS)))
    cases_u8.append(("empty", b""))
    cases_u16.append(("empty", b""))
    for k, (data, _off) in enumerate(T.UTF8_ERROR_CASES):
        cases_u8.append((f"error-{k}", data))
    for k, (data, _off) in enumerate(T.UTF16_ERROR_CASES):
        cases_u16.append((f"error-{k}", data))

    rng = random.Random(20221209)
    # arbitrary bytes, biased towards the interesting lead/continuation ranges
    interesting = list(range(0x80, 0x100)) + [0x00, 0x20, 0x41, 0x7F]
    for k in range(600):
        n = rng.randrange(0, 72)
        if k % 2:
            data = bytes(rng.choice(interesting) for _ in range(n))
        else:
            data = bytes(rng.randrange(256) for _ in range(n))
        cases_u8.append((f"random-{k}", data))
    # surrogate soup and arbitrary words
    soup = [0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0xD835, 0xDCAA, 0x0041, 0x00E9, 0x4E2D, 0xFFFF, 0x007F, 0x0080, 0x07FF, 0x0800]
    for k in range(600):
        n = rng.randrange(0, 48)
        if k % 2:
            words = [rng.choice(soup) for _ in range(n)]
        else:
            words = [rng.randrange(0x10000) for _ in range(n)]
        cases_u16.append((f"random-{k}", words_to_bytes(words)))

    # corpus-generated valid text (every script class) plus one-error mutations
    for cls in corpus.SCRIPT_CLASSES:
        for size, seed in ((200, 1), (3000, 2), (20000, 3)):
            mutate_here = size <= 3000
            utf8, utf16 = corpus.generate(corpus.CorpusSpec(cls, size, seed=seed))
            cases_u8.append((f"corpus-{cls}-{size}", utf8))
            cases_u16.append((f"corpus-{cls}-{size}", utf16))
            if not mutate_here:
                continue
            for j, ecls in enumerate(corpus.UTF8_ERROR_CLASSES):
                for strat in corpus.POSITION_STRATEGIES:
                    try:
                        mutated, _ = corpus.mutate(
                            utf8, corpus.ErrorRecipe(ecls, strat), seed=seed * 100 + j
                        )
                    except corpus.RecipeNotApplicable:
                        continue
                    cases_u8.append((f"mutated-{cls}-{size}-{ecls}-{strat}", mutated))
            for j, ecls in enumerate(corpus.UTF16_ERROR_CLASSES):
                for strat in corpus.POSITION_STRATEGIES:
                    try:
                        mutated, _ = corpus.mutate(
                            utf16, corpus.ErrorRecipe(ecls, strat), seed=seed * 100 + j
                        )
                    except corpus.RecipeNotApplicable:
                        continue
                    cases_u16.append((f"mutated-{cls}-{size}-{ecls}-{strat}", mutated))

    golden = {
        "generator": "tests/golden/make_golden.py",
        "reference": "laneutf 0.1.0 scalar (pkg/src/laneutf/scalar.py)",
        "utf8_to_utf16": [],
        "utf16_to_utf8": [],
    }
    for name, data in cases_u8:
        outcome, payload = scalar.transcode_utf8_to_utf16le(data)
        v = scalar.validate_utf8(data)
        golden["utf8_to_utf16"].append(
            {
                "name": name,
                "input": b64(data),
                "outcome": outcome_tuple(outcome),
                "payload": payload_field(payload),
                "validate": outcome_tuple(v),
            }
        )
    for name, data in cases_u16:
        outcome, payload = scalar.transcode_utf16le_to_utf8(data)
        v = scalar.validate_utf16le(data)
        golden["utf16_to_utf8"].append(
            {
                "name": name,
                "input": b64(data),
                "outcome": outcome_tuple(outcome),
                "payload": payload_field(payload),
                "validate": outcome_tuple(v),
            }
        )

    # frozen offsets from the reference test module (test_scalar.py:84-121)
    golden["utf8_error_offsets"] = [[b64(d), off] for d, off in T.UTF8_ERROR_CASES]
    golden["utf16_error_offsets"] = [[b64(d), off] for d, off in T.UTF16_ERROR_CASES]

    # every byte pair: consumed of scalar.validate_utf8 (exhaustive 2-byte sweep)
    pairs = bytearray(65536)
    for i in range(65536):
        pairs[i] = scalar.validate_utf8(bytes((i & 0xFF, i >> 8))).consumed
    golden["utf8_pair_consumed"] = b64(bytes(pairs))

    # SplitMix64 streams (corpus.py:65-82)
    streams = {}
    for seed in (0, 1, 7, 123456789, (1 << 64) - 1):
        r = corpus.SplitMix64(seed)
        streams[str(seed)] = [format(r.next_u64(), "016x") for _ in range(64)]
    golden["splitmix64"] = streams

    path = os.path.join(HERE, "golden.json.gz")
    with gzip.open(path, "wt", compresslevel=9) as fh:
        json.dump(golden, fh, separators=(",", ":"))
    print(f"wrote {path}: {len(cases_u8)} utf8 cases, {len(cases_u16)} utf16 cases, "
          f"{os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
