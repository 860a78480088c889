"""Native UCR text parsing (ek_parse_tsv via ingest.load_tsv_packed) against the
reference-semantics loader (series.load_tsv, pkg/src/elastik/series.py:61-86): the same
labels, values (bit-for-bit) and errors, including the files the fast path hands back.
Mirrors the reference's tests (pkg/tests/test_series.py:18-91).  Host only: no device."""

import numpy as np
import pytest

from paper_2102_05221_b200 import ingest, series
from paper_2102_05221_b200.errors import EmptyDatasetError, ParseError


def _both(tmp_path, text, delimiter="tab", binary=False):
    p = tmp_path / "d.tsv"
    if binary:
        p.write_bytes(text)
    else:
        p.write_bytes(text.encode("utf-8"))
    got = exc_got = want = exc_want = None
    try:
        got = ingest.load_tsv_packed(p, delimiter=delimiter, pinned=False)
    except Exception as e:  # noqa: BLE001
        exc_got = e
    try:
        want = series.load_tsv(p, delimiter=delimiter)
    except Exception as e:  # noqa: BLE001
        exc_want = e
    if exc_want is not None:
        assert exc_got is not None and type(exc_got) is type(exc_want) and str(exc_got) == str(exc_want)
        return None
    assert exc_got is None, exc_got
    assert list(got.labels) == want.labels
    assert len(got) == len(want)
    for s, (_, v) in enumerate(want.entries):
        assert np.array_equal(got.series(s), v) and got.series(s).tobytes() == v.tobytes()
    return got


@pytest.mark.parametrize("text", [
    "1\t1.5\t2\t-3e-2\n",
    "1\t1.5\t2\r\n2\t3\t4\r\n",                 # CRLF
    "1\t1\r2\t2\r",                            # lone CR ends a line (universal newlines)
    "\n\n1\t1\n \t \n\x0c\n2\t2\n\n",          # blank and whitespace-only lines
    "3.7\t1\n-2.9\t2\n+0.5\t3\n-0\t4\n",       # labels truncate toward zero
    "1\t.5\t5.\t+7E+1\t-1e-300\t 2 \t1e308\n",  # decimal forms, padding, extremes
    "1\t0.1\t0.2\t0.30000000000000004\t123456789012345678901234567890\n",
    "1\t4.9406564584124654e-324\t2.2250738585072014e-308\n",  # subnormals
])
def test_fast_path_matches_reference(tmp_path, text):
    assert _both(tmp_path, text) is not None


def test_comma_delimiter(tmp_path):
    assert _both(tmp_path, "1,1.5,2\n2,3,4\n", delimiter="comma") is not None
    _both(tmp_path, "1\t1.5\t2\n", delimiter="comma")  # one field per line under comma: same error


@pytest.mark.parametrize("text", [
    "1\t1_0\t2\n",          # underscores: float() accepts them (fallback decides)
    "1\tinf\t2\n",          # non-finite
    "1\tnan\n",
    "1\t1e999\n",           # overflow to inf
    "1\tx\t2\n",            # not a number
    "1\t\t2\n",             # empty field
    "7\n",                  # a label without values
    "",                     # empty file
    "\n \n",                # only blank lines
    "1\t1\n2\t0x10\n",      # hex is not a Python float literal
    "1\t١٢\n",    # non-ASCII digits (float() accepts Arabic-Indic digits)
    "﻿1\t2\n",         # a BOM stays part of the first field under utf-8
    "1e30\t1\n",            # a label beyond int64 is still an int in Python
])
def test_fallback_cases_match_reference(tmp_path, text):
    _both(tmp_path, text)


def test_invalid_utf8_is_the_reference_error(tmp_path):
    _both(tmp_path, b"1\t2\xff\n", binary=True)


def test_error_positions(tmp_path):
    p = tmp_path / "e.tsv"
    p.write_text("1\t2\t3\n2\t4\tabc\n")
    with pytest.raises(ParseError) as ei:
        ingest.load_tsv_packed(p, pinned=False)
    assert ei.value.line == 2 and ei.value.column == 3
    p.write_text("")
    with pytest.raises(EmptyDatasetError):
        ingest.load_tsv_packed(p, pinned=False)


def test_round_trip_random(tmp_path, rng):
    entries = []
    for k in range(60):
        n = int(rng.integers(1, 300))
        entries.append((int(rng.integers(-5, 50)), rng.normal(scale=10.0 ** rng.integers(-8, 9), size=n)))
    ds = series.LabeledDataset("r", tuple(entries))
    p = tmp_path / "r.tsv"
    series.write_tsv(ds, p)
    got = ingest.load_tsv_packed(p, pinned=False)
    for s, (lab, v) in enumerate(entries):
        assert got.labels[s] == lab and got.series(s).tobytes() == v.tobytes()
    back = got.to_labeled()
    assert [e[0] for e in back.entries] == [e[0] for e in entries]
