"""The EXCE edit-log format and the reference decoder (CPU): SPEC's
apply_edit_log examples on hand-built streams."""
import struct

import numpy as np
import pytest

import edit_log_ref as R


def varint(v):
    out = bytearray()
    while v >= 0x80:
        out.append((v & 0x7F) | 0x80)
        v >>= 7
    out.append(v)
    return bytes(out)


def stream(xi, N, dims, entries):
    body = bytearray()
    prev = -1
    for i, k, v in entries:
        body += varint(i - prev - 1)
        prev = i
        body.append(k)
        if k == 0:
            body += np.float32(v).tobytes()
    h = R.HEADER.pack(b"EXCE", 1, 0, 0, xi, N, *dims, len(entries), len(body), len(body))
    return h + bytes(body)


def test_empty_log_is_identity():
    g = np.arange(6, dtype=np.float32)
    d = R.parse(stream(0.5, 5, (6, 1, 1), []))
    assert np.array_equal(R.apply(g, d), g)


def test_stepped_two_with_xi_half():
    # Stepped(2), xi = 0.5, N = 5 -> decreased by 2 Delta = 0.2 (two
    # float32 steps of RN(0.5 / 5))
    g = np.array([1.0, 3.0, 7.0], np.float32)
    d = R.parse(stream(0.5, 5, (3, 1, 1), [(1, 2, None)]))
    out = R.apply(g, d)
    delta = np.float32(np.float32(0.5) / np.float32(5))
    assert out[1] == np.float32(np.float32(3.0 - delta) - delta)
    assert abs(float(out[1]) - 2.8) < 1e-6 and out[0] == 1.0 and out[2] == 7.0


def test_lossless_value_and_gaps():
    # a Lossless entry stores f_v - xi exactly; index gaps across varint bytes
    g = np.zeros(300, np.float32)
    d = R.parse(stream(1.0, 5, (300, 1, 1), [(0, 0, -0.75), (129, 1, None), (299, 0, 2.5)]))
    out = R.apply(g, d)
    assert out[0] == np.float32(-0.75) and out[299] == np.float32(2.5)
    assert out[129] == np.float32(0 - np.float32(0.2))
    assert [e[0] for e in d["entries"]] == [0, 129, 299]


def test_truncated_stream_is_rejected():
    s = stream(1.0, 5, (10, 1, 1), [(3, 0, 1.0)])
    with pytest.raises(Exception):
        R.parse(s[:-1])
