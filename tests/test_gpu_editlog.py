"""NEXT-4: the edit set E as a compact log (exactz_edit_log,
P:245).  Round trip through the GPU encoder and the
GPU apply, and through an independent Python decoder of the byte format."""
import ctypes

import numpy as np
import pytest
import torch

import edit_log_ref as R
from synth import fields as S

pytestmark = pytest.mark.gpu


def zstd_decompress(body: bytes, raw: int) -> bytes:
    z = ctypes.CDLL("libzstd.so.1")
    z.ZSTD_decompress.restype = ctypes.c_size_t
    out = ctypes.create_string_buffer(raw)
    n = z.ZSTD_decompress(out, raw, body, len(body))
    assert n == raw
    return out.raw


@pytest.mark.parametrize("cfg,shape,mode,level", [("C1", None, "uniform", 0),
                                                  ("C1", None, "sz", 3),
                                                  ("C2", (30, 20, 70), "uniform", 0),
                                                  ("C3", (24, 19, 66), "uniform", 5)])
def test_edit_log_round_trip(exactz, cfg, shape, mode, level):
    f, g, xi = S.make(cfg, shape=shape, mode=mode)
    fd, gd = f.cuda(), g.cuda()
    c = torch.empty(f.numel(), dtype=torch.uint8, device="cuda")
    r = exactz.exactz_correct(fd, gd, xi, edit_counts=c)
    assert r.status == 0
    log, ne = exactz.exactz_edit_log(gd, r.out, c, xi, level=level)
    cn = c.cpu().numpy()
    assert ne == int((cn > 0).sum())
    # GPU apply: the corrected field, bit for bit
    back = exactz.exactz_edit_log_apply(log, gd)
    assert torch.equal(back.view(torch.int32), r.out.view(torch.int32))
    # independent decoder: same field; Stepped(k) carries the edit count
    d = R.parse(log, zstd_decompress)
    assert d["N"] == 5 and len(d["entries"]) == ne
    ref = R.apply(g.numpy(), d)
    assert np.array_equal(ref.view(np.uint32), r.out.cpu().numpy().view(np.uint32))
    for i, k, v in d["entries"]:
        if k:
            assert cn[i] == k
    # stepped entries never undershoot lo ("corruption error" otherwise)
    lo = (f.double() - xi).numpy().reshape(-1)
    assert (ref.reshape(-1).astype(np.float64) >= lo - 1e-6).all()


def test_edit_log_empty_and_malformed(exactz):
    f, _, xi = S.make("C1")
    fd = f.cuda()
    c = torch.zeros(f.numel(), dtype=torch.uint8, device="cuda")
    log, ne = exactz.exactz_edit_log(fd, fd, c, xi)
    assert ne == 0 and len(log) == 64
    assert torch.equal(exactz.exactz_edit_log_apply(log, fd), fd)
    bad = b"EXCX" + log[4:]
    assert exactz.status_of(exactz.exactz_edit_log_apply, bad, fd) == exactz.EINVAL
    g = S.decompress(f, xi, seed=5).cuda()
    c2 = torch.empty(f.numel(), dtype=torch.uint8, device="cuda")
    r = exactz.exactz_correct(fd, g, xi, edit_counts=c2)
    log, ne = exactz.exactz_edit_log(g, r.out, c2, xi)
    assert ne > 0
    truncated = log[:-1]
    assert exactz.status_of(exactz.exactz_edit_log_apply, truncated, g) == exactz.EINVAL


def test_edit_log_untrusted_streams(exactz):
    """a varint gap >= 2^63, a payload size that wraps the header
    sum, and a header whose dims disagree with the caller's buffers are all
    EXACTZ_EINVAL, before any device write."""
    import struct
    f, _, xi = S.make("C1")
    fd = f.cuda()
    c = torch.zeros(f.numel(), dtype=torch.uint8, device="cuda")
    hdr, _ = exactz.exactz_edit_log(fd, fd, c, xi)
    assert len(hdr) == 64
    E = exactz

    def with_payload(pay, entries):
        h = bytearray(hdr)
        struct.pack_into("<QQQ", h, 40, entries, len(pay), len(pay))
        return bytes(h) + pay

    # one entry whose gap is 2^63 + 5 (10-byte varint), kind Stepped(1)
    gap = (1 << 63) + 5
    vb = bytearray()
    while True:
        b = gap & 0x7F
        gap >>= 7
        vb.append(b | (0x80 if gap else 0))
        if not gap:
            break
    out = fd.clone()
    assert E.status_of(E.exactz_edit_log_apply, with_payload(bytes(vb) + b"\x01", 1), fd,
                       out=out) == E.EINVAL
    assert torch.equal(out, fd)
    # gap exactly past the end: V (index V), and V - 1 (the last vertex) is fine
    V = f.numel()
    for gap, ok in ((V, False), (V - 1, True)):
        vb = bytearray()
        while True:
            b = gap & 0x7F
            gap >>= 7
            vb.append(b | (0x80 if gap else 0))
            if not gap:
                break
        st = E.status_of(E.exactz_edit_log_apply, with_payload(bytes(vb) + b"\x01", 1), fd)
        assert (st == E.OK) == ok
    # payload size near 2^64: the header sum would wrap
    h = bytearray(hdr)
    struct.pack_into("<QQQ", h, 40, 0, (1 << 64) - 32, (1 << 64) - 32)
    assert E.status_of(E.exactz_edit_log_apply, bytes(h), fd) == E.EINVAL
    # dims of the stream (16^3) against a smaller caller buffer
    assert E.status_of(E.exactz_edit_log_apply, hdr, fd[:8].contiguous()) == E.EINVAL
