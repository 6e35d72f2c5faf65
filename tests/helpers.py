"""Small helpers shared by the test modules."""

import base64
import hashlib


def payload_matches(field: str, payload: bytes) -> bool:
    """Golden payload fields are base64 (small) or 'sha256:<hex>' (large)."""
    if field.startswith("sha256:"):
        return hashlib.sha256(payload).hexdigest() == field[7:]
    return base64.b64decode(field) == payload


def words_to_bytes(words):
    return b"".join(int(w).to_bytes(2, "little") for w in words)
