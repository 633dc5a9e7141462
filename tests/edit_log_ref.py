"""Reference decoder of the EXCE edit log (test infrastructure, independent
of the CUDA path): plain Python over the byte format of
paper_2604_01397_b200/csrc/editlog.cuh and include/exactz.h, with the
SPEC apply_edit_log semantics: Stepped(k) replays k steps
RN_f32(g - Delta) from g^, Delta = RN_f32(xi / N); Lossless stores the value."""
import struct

import numpy as np

HEADER = struct.Struct("<4sBBHfIqqqQQQ")  # 64 bytes


def parse(log: bytes, decompress=None):
    magic, ver, codec, _r, xi, N, nx, ny, nz, ne, pay, raw = HEADER.unpack_from(log, 0)
    assert magic == b"EXCE" and ver == 1 and HEADER.size == 64
    body = log[64:64 + pay]
    if codec == 1:
        body = decompress(body, raw)
    assert len(body) == raw
    entries, p, prev = [], 0, -1
    for _ in range(ne):
        d, sh = 0, 0
        while True:
            b = body[p]
            p += 1
            d |= (b & 0x7F) << sh
            sh += 7
            if not b & 0x80:
                break
        i = prev + 1 + d
        prev = i
        k = body[p]
        p += 1
        v = None
        if k == 0:
            v = np.frombuffer(body[p:p + 4], dtype=np.float32)[0]
            p += 4
        entries.append((i, k, v))
    assert p == len(body)
    return dict(xi=np.float32(xi), N=N, dims=(nx, ny, nz), entries=entries)


def apply(ghat: np.ndarray, log: dict) -> np.ndarray:
    g = ghat.reshape(-1).astype(np.float32).copy()
    delta = np.float32(log["xi"] / np.float32(log["N"]))
    for i, k, v in log["entries"]:
        if k == 0:
            g[i] = v
        else:
            t = np.float32(g[i])
            for _ in range(k):
                t = np.float32(t - delta)
            g[i] = t
    return g.reshape(ghat.shape)
