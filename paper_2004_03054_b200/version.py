"""Job-side data types of the compaction path (mirrors, not the MANIFEST).

Only what crosses the compaction boundary is mirrored here:

* ``SstMeta``        — ``pkg/src/luda/sst.py:52-64``
* ``Version``        — ``pkg/src/luda/version.py:96-128`` (levels + ``covers_below``)
* ``CompactionJob``  — ``pkg/src/luda/version.py:146-159``

``run_compaction`` duck-types its ``job`` argument, so the reference's own
``CompactionJob``/``Version`` objects can be passed in unchanged. The MANIFEST /
``VersionSet`` machinery is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field

NUM_LEVELS = 7
TRAILER_SIZE = 8


def user_key_of(ikey: bytes) -> bytes:
    return ikey[:-TRAILER_SIZE]


@dataclass
class SstMeta:
    file_id: int
    file_size: int
    smallest: bytes
    largest: bytes
    level: int = 0

    def overlaps(self, lo_user: bytes, hi_user: bytes) -> bool:
        return user_key_of(self.smallest) <= hi_user and user_key_of(self.largest) >= lo_user


class Version:
    """Per-level file lists; only ``covers_below`` matters to compaction."""

    __slots__ = ("levels", "refs")

    def __init__(self, levels=None):
        self.levels = levels if levels is not None else [[] for _ in range(NUM_LEVELS)]
        self.refs = 0

    @classmethod
    def empty(cls) -> "Version":
        return cls()

    def covers_below(self, user_key: bytes, level: int) -> bool:
        for deeper in range(level + 1, len(self.levels)):
            for f in self.levels[deeper]:
                if user_key_of(f.smallest) <= user_key <= user_key_of(f.largest):
                    return True
        return False


@dataclass
class CompactionJob:
    source_level: int
    lower: list
    upper: list
    target_level: int
    version: Version
    grandparents: list = field(default_factory=list)

    def input_files(self):
        return self.lower + self.upper

    def input_bytes(self) -> int:
        return sum(f.file_size for f in self.input_files())


def deeper_ranges(version, target_level: int):
    """User-key intervals of every file below ``target_level``.

    This is the data behind ``Version.covers_below`` (version.py:122-128): a
    key is covered iff it lies in one of these closed intervals. Returned
    sorted and merged so the device can binary-search them.
    """
    spans = []
    levels = getattr(version, "levels", None) or []
    for deeper in range(target_level + 1, len(levels)):
        for f in levels[deeper]:
            lo, hi = user_key_of(f.smallest), user_key_of(f.largest)
            if lo <= hi:
                spans.append((lo, hi))
    spans.sort()
    merged = []
    for lo, hi in spans:
        if merged and lo <= merged[-1][1]:
            if hi > merged[-1][1]:
                merged[-1] = (merged[-1][0], hi)
        else:
            merged.append((lo, hi))
    return merged
