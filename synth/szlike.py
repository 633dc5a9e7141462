"""SZ-like base compressor for the overall-compression-ratio report (SURVEY
§8(f) NEXT-4: "OCR against an SZ-like synthetic compressor"; P:433 defines
OCR as the original size over the compressed size plus the stored edits).

This is NOT part of EXaCTz: it is a stand-in for the error-bounded lossy
compressor whose decompressed output ghat the correction repairs, so that the
edit log can be sized against a base stream.  It encodes exactly the field
`fields.decompress(f, xi, seed, mode="sz")` produces:

  q      = round(f / 2 xi)           (float64, as the generator; int64)
  r      = the 3D Lorenzo residual of q: mixed first differences along x, y
           and z with zeros outside the grid (SZ's 1-layer Lorenzo predictor
           applied to the quantisation codes)
  codes  = zigzag(r) as one byte when < 255, else 255 and the value in an
           escape stream (u32)
  exc    = the vertices where ghat != RN_f32(2 xi q) (the generator's
           one-ulp nudges into [f - xi, f + xi]): index deltas and values
  stream = zstd level 3 of codes, escapes, exc (pyarrow's codec)

`decode` inverts it (prefix sums along z, y, x; RN_f32(2 xi q); exceptions)
and is checked bit for bit against the generator in tests/test_synth.py.
"""
import numpy as np
import pyarrow as pa
import torch

_HEADER = 64  # magic, version, xi, shape, stream lengths


def _zstd(a: np.ndarray, level: int = 3) -> bytes:
    return pa.Codec("zstd", compression_level=level).compress(np.ascontiguousarray(a),
                                                                asbytes=True)


def _unzstd(b: bytes, nbytes: int) -> np.ndarray:
    return np.frombuffer(pa.Codec("zstd").decompress(b, decompressed_size=nbytes, asbytes=True),
                         dtype=np.uint8)


def _lorenzo(q: torch.Tensor) -> torch.Tensor:
    r = q
    for d in range(q.dim()):
        r = torch.diff(r, dim=d, prepend=torch.zeros_like(r.narrow(d, 0, 1)))
    return r


def encode(f: torch.Tensor, xi: float, ghat: torch.Tensor, level: int = 3) -> dict:
    """Streams and sizes of ghat (= decompress(f, xi, mode="sz")) as above."""
    xi = float(np.float32(xi))
    q = torch.round(f.to(torch.float64) / (2 * xi)).to(torch.int64)
    r = _lorenzo(q).reshape(-1)
    z = (r << 1) ^ (r >> 63)  # zigzag
    codes = torch.where(z < 255, z, torch.full_like(z, 255)).to(torch.uint8)
    esc = z[z >= 255]
    assert bool((esc < 2 ** 32).all())
    base = (2 * xi * q.to(torch.float64)).to(torch.float32).reshape(-1)
    gh = ghat.reshape(-1)
    exc = torch.nonzero(gh.view(torch.int32) != base.view(torch.int32)).reshape(-1)
    codes_h = codes.cpu().numpy()
    esc_h = esc.to(torch.int64).cpu().numpy().astype(np.uint32)
    exc_i = exc.cpu().numpy().astype(np.int64)
    exc_d = np.diff(exc_i, prepend=np.int64(-1)).astype(np.int64)
    exc_v = gh[exc].cpu().numpy().view(np.uint32)
    s_codes, s_esc = _zstd(codes_h, level), _zstd(esc_h, level)
    s_exc = _zstd(np.concatenate([exc_d.view(np.uint8), exc_v.view(np.uint8)]), level)
    nbytes = _HEADER + len(s_codes) + len(s_esc) + len(s_exc)
    return {"shape": tuple(f.shape), "xi": xi, "n": int(codes_h.size), "n_esc": int(esc_h.size),
            "n_exc": int(exc_i.size), "codes": s_codes, "esc": s_esc, "exc": s_exc,
            "bytes": nbytes}


def decode(enc: dict) -> torch.Tensor:
    """ghat from the streams (CPU, float32)."""
    n, ne, nx = enc["n"], enc["n_esc"], enc["n_exc"]
    codes = _unzstd(enc["codes"], n).astype(np.int64)
    esc = _unzstd(enc["esc"], 4 * ne).view(np.uint32).astype(np.int64) if ne else np.zeros(0, np.int64)
    z = codes.copy()
    z[codes == 255] = esc
    r = (z >> 1) ^ -(z & 1)  # un-zigzag
    q = torch.from_numpy(r).reshape(enc["shape"])
    for d in range(q.dim()):
        q = torch.cumsum(q, dim=d)
    g = (2 * enc["xi"] * q.to(torch.float64)).to(torch.float32).reshape(-1)
    if nx:
        ex = _unzstd(enc["exc"], 12 * nx)
        idx = np.cumsum(ex[:8 * nx].view(np.int64)) - 1  # deltas from index -1
        val = ex[8 * nx:].view(np.uint32).view(np.float32)
        g[torch.from_numpy(idx)] = torch.from_numpy(val.copy())
    return g.reshape(enc["shape"])
