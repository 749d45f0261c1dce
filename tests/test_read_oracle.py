"""Pin the oracle's read-path restatement (MemTable / BlockReader / store_get,
oracle/luda_oracle.py) against the reference's own Table.get results frozen by
tests/golden/make_golden.py (tests/golden/reads.json). CPU-only."""

import hashlib
import json
import os

import pytest

from oracle import luda_oracle as O
from tests.golden import read_cases as RC

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "reads.json")))


def oracle_outcomes(c):
    tables = [O.MemTable(f) for f in c["files"]]
    enc = []
    for t, q in c["queries"]:
        if c["mode"] == "table":
            o = RC.outcome(lambda: tables[t].get(q))
        else:
            o = RC.outcome(lambda: O.store_get(tables, c["l0"], c["levels"], q))
        enc.append(RC.encode(c["mode"], o))
    return enc, [[tb.filter_rejects, tb.data_block_reads] for tb in tables]


@pytest.mark.parametrize("name", RC.READ_CASES)
def test_read_oracle_matches_reference(name):
    c = RC.build(name)
    g = GOLD[name]
    assert [hashlib.sha256(f).hexdigest() for f in c["files"]] == g["files"]
    enc, counters = oracle_outcomes(c)
    assert RC.summary(enc) == g["results"]
    assert counters == g["counters"]


def test_read_cases_cover_the_error_paths():
    """The malformed and corrupt cases reach every Table.get failure class."""
    kinds = set()
    for name in ("malformed", "corrupt"):
        enc, _ = oracle_outcomes(RC.build(name))
        kinds |= {tuple(e[:2]) for e in enc if e is not None and e[0] == "E"}
    assert ("E", "CorruptionError") in kinds
    assert ("E", "FormatError") in kinds
    assert ("E", "struct.error") in kinds
