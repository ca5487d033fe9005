"""The oracle's parse restatement (oracle.parse_line, Fe:175-235) against the
reference's own parse_example outputs (tests/golden/parse.npz): which lines
raise, labels, canonical (field, index, value) -- bit for bit.  CPU only."""

import numpy as np

from oracle import fieldwise_oracle as fo
from paper_2407_10115_b200.features import InputSchema, split_lines
from tests.golden_io import load


def golden_lines():
    g = load("parse")
    buf, off = split_lines(g["text"])
    lines = [bytes(buf[off[i]:off[i + 1]]).rstrip(b"\n") for i in range(len(off) - 1)]
    return g, lines, InputSchema.from_text(str(g["schema"]))


def test_oracle_parse_matches_reference_golden():
    g, lines, sc = golden_lines()
    ok, labels, off, cnt, idx, val = fo.parse_lines_ragged(lines, sc.field_names,
                                                           sc.numeric_fields, sc.hash_bits)
    assert np.array_equal(ok, g["ok"])
    assert np.array_equal(labels[ok], g["labels"][ok])
    assert np.array_equal(off, g["ex_off"])
    assert np.array_equal(idx, g["idx"])
    assert np.array_equal(val.view(np.uint64), g["val"].view(np.uint64))
    fid = np.repeat(np.tile(np.arange(sc.n_fields), len(lines)), cnt.ravel())
    assert np.array_equal(fid, g["fid"])


def test_schema_text_round_trip_and_contract():
    sc = InputSchema(("a", "b"), frozenset({"b"}), 20)
    assert InputSchema.from_text(sc.to_text()).to_text() == sc.to_text()
    import pytest
    from paper_2407_10115_b200.errors import ParseError
    with pytest.raises(ParseError):
        InputSchema(("a", "a"))
    with pytest.raises(ParseError):
        InputSchema(("a",), hash_bits=30)
    with pytest.raises(ParseError):
        InputSchema(("a",), frozenset({"b"}))


def test_split_lines_offsets():
    buf, off = split_lines(b"1 |a x\n\n0 |b y")
    assert off.tolist() == [0, 7, 8, 14]
    buf, off = split_lines(b"1 |a x\n")
    assert off.tolist() == [0, 7]
    buf, off = split_lines(b"")
    assert off.tolist() == [0]
