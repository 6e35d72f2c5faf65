"""Result types of the transcoding entry points.

Mirrors ``laneutf.outcome`` (/root/reference/pkg/src/laneutf/outcome.py:51-83)
so callers of the reference read results the same way: ``status`` is a
``TranscodeStatus`` with the same string values, ``consumed`` counts input
code units strictly before the first invalid unit (so it doubles as the error
offset) and ``written`` counts output code units.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

__all__ = ["TranscodeStatus", "TranscodeOutcome", "STATUS_BY_CODE"]


class TranscodeStatus(enum.Enum):
    OK = "ok"
    MALFORMED_INPUT = "malformed-input"
    OUTPUT_TOO_SMALL = "output-too-small"


# numeric codes of lu_outcome.status (include/laneutf_b200.h)
STATUS_BY_CODE = {
    0: TranscodeStatus.OK,
    1: TranscodeStatus.MALFORMED_INPUT,
    2: TranscodeStatus.OUTPUT_TOO_SMALL,
}


@dataclass(frozen=True)
class TranscodeOutcome:
    """What a transcoding call did (outcome.py:57-83).

    ``consumed`` and ``written`` count code units of the input and output
    encodings (bytes for UTF-8, 16-bit words for UTF-16).
    """

    status: TranscodeStatus
    consumed: int
    written: int

    @property
    def ok(self) -> bool:
        return self.status is TranscodeStatus.OK

    @property
    def error_offset(self) -> int:
        """Offset of the first rejected input unit (MALFORMED_INPUT only)."""
        if self.status is not TranscodeStatus.MALFORMED_INPUT:
            raise ValueError(f"no error offset for status {self.status.value!r}")
        return self.consumed

    def as_tuple(self) -> tuple[str, int, int]:
        """(status value, consumed, written): comparable across packages."""
        return (self.status.value, self.consumed, self.written)
