"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the tests, bench.py and smoke(): it serves the oracle
and the CUDA path with identical bytes.  It holds NONE of the method's
arithmetic (no SoS, no classification, no edits); it only makes fields.

Arrays are float32 of shape (nz, ny, nx) (x fastest), i.e. the linear index is
x + nx*(y + ny*z) as in the C-ABI (include/exactz.h).

Generators (BASELINE.json configs):
  gaussmix      16^3 sum of Gaussians, mixed signs (config C1)
  nyx_like      log-normal Gaussian random field, P(k) ~ k^-2 exp(-(k/kc)^2)
                (cosmology density; NYX) (configs C2, C5)
  combustion    flame-sheet temperature from a Kolmogorov-spectrum mixture
                fraction (Combustion 560^3) (config C3)
  climate2d     zonal-mean temperature + GRF anomalies, 3600x1800 (config C4)
Simulated decompression (BASELINE.json "uniform quantisation noise at relative
eps"): ghat_i = RN_f32(f_i + xi*u_i) with u_i from a counter-based splitmix64,
nudged by whole ulps until |ghat_i - f_i| <= xi holds exactly.
"""
from __future__ import annotations

import math

import numpy as np
import torch

GOLDEN = 0x9E3779B97F4A7C15


def _i64(x: int) -> int:
    """reinterpret a uint64 constant as int64 (torch has no uint64 arithmetic)"""
    return x - (1 << 64) if x >= (1 << 63) else x


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    """logical right shift of int64 bit patterns"""
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(z: torch.Tensor) -> torch.Tensor:
    z = z + _i64(GOLDEN)
    z = (z ^ _srl(z, 30)) * _i64(0xBF58476D1CE4E5B9)
    z = (z ^ _srl(z, 27)) * _i64(0x94D049BB133111EB)
    return z ^ _srl(z, 31)


def uniform_pm1(n: int, seed: int, device="cpu", start: int = 0) -> torch.Tensor:
    """u_i = 2*(splitmix64(seed*GOLDEN ^ i) >> 11) * 2^-53 - 1 in [-1, 1), float64.

    Counter-based: identical on any host/device for a given (seed, i)."""
    key = _i64((seed * GOLDEN) % (1 << 64))
    idx = torch.arange(start, start + n, dtype=torch.int64, device=device)
    r = splitmix64(idx ^ key)
    return _srl(r, 11).to(torch.float64) * (2.0 ** -53) * 2.0 - 1.0


def _kgrid(shape, device):
    """|k| in cycles/sample for an rfftn layout of `shape`"""
    ks = [torch.fft.fftfreq(n, device=device, dtype=torch.float64) for n in shape[:-1]]
    ks.append(torch.fft.rfftfreq(shape[-1], device=device, dtype=torch.float64))
    k2 = None
    for ax, k in enumerate(ks):
        view = [1] * len(shape)
        view[ax] = k.numel()
        term = (k.view(view)) ** 2
        k2 = term if k2 is None else k2 + term
    return torch.sqrt(k2)


def grf(shape, spectrum, seed: int, device="cpu") -> torch.Tensor:
    """Unit-variance Gaussian random field with power spectrum P(|k|) (float64)."""
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    w = torch.randn(shape, generator=gen, dtype=torch.float64, device=device)
    W = torch.fft.rfftn(w)
    del w
    k = _kgrid(shape, device)
    amp = torch.sqrt(spectrum(torch.where(k > 0, k, torch.ones_like(k))))
    amp = torch.where(k > 0, amp, torch.zeros_like(amp))
    del k
    W *= amp
    del amp
    d = torch.fft.irfftn(W, s=shape)
    del W
    d -= d.mean()
    d /= d.std()
    return d


def xi_from_rel(f32: torch.Tensor, rel: float) -> float:
    """xi = RN_f32(rel * (max f - min f)), computed in double (amb-19)."""
    rng = float(f32.max().double() - f32.min().double())
    return float(np.float32(rel * rng))


def _shift_min_to(f64: torch.Tensor, rel: float) -> torch.Tensor:
    """Offset rule: uniform shift so that min f >= xi."""
    rng = float(f64.max() - f64.min())
    xi = rel * rng
    lo = float(f64.min())
    if lo < 1.01 * xi:
        f64 = f64 + (1.01 * xi - lo)
    return f64


def gaussmix(n: int = 16, K: int = 8, seed: int = 1, rel: float = 1e-2, device="cpu"):
    """f(p) = 2 + sum_k a_k exp(-|p-c_k|^2 / (2 sigma_k^2)), c ~ U[0,n)^3,
    sigma ~ U[1.5,4], a ~ U[-1,1]."""
    rs = np.random.default_rng(seed)
    c = rs.uniform(0, n, size=(K, 3))
    s = rs.uniform(1.5, 4.0, size=K)
    a = rs.uniform(-1.0, 1.0, size=K)
    z, y, x = torch.meshgrid(*[torch.arange(n, dtype=torch.float64, device=device)] * 3,
                             indexing="ij")
    f = torch.full((n, n, n), 2.0, dtype=torch.float64, device=device)
    for k in range(K):
        r2 = (x - c[k, 0]) ** 2 + (y - c[k, 1]) ** 2 + (z - c[k, 2]) ** 2
        f += a[k] * torch.exp(-r2 / (2 * s[k] ** 2))
    return _shift_min_to(f, rel).to(torch.float32)


def nyx_like(shape=(512, 512, 512), seed: int = 2, rel: float = 1e-3, sigma: float = 1.5,
             device="cpu"):
    """Log-normal density rho = exp(sigma*delta - sigma^2/2), delta a GRF with
    P(k) ~ k^-2 exp(-(k/kc)^2), kc = k_Nyquist/4; f = rho + xi (offset rule)."""
    kc = 0.5 / 4.0
    d = grf(shape, lambda k: k ** -2.0 * torch.exp(-(k / kc) ** 2), seed, device)
    d.mul_(sigma).sub_(sigma * sigma / 2).exp_()
    rng = float(d.max() - d.min())
    d += rel * rng
    return d.to(torch.float32)


def combustion(shape=(560, 560, 560), seed: int = 3, rel: float = 1e-4, device="cpu"):
    """Mixture fraction Z = (1 + tanh(G/0.3))/2, G a GRF with P(k) ~ k^-11/3;
    temperature f = 300 + 1700 exp(-((Z-0.3)/0.1)^2) K (thin flame sheets)."""
    g = grf(shape, lambda k: k ** (-11.0 / 3.0), seed, device)
    g.div_(0.3).tanh_().add_(1.0).mul_(0.5)          # Z
    g.sub_(0.3).div_(0.1).square_().neg_().exp_()    # exp(-((Z-0.3)/0.1)^2)
    g.mul_(1700.0).add_(300.0)
    return _shift_min_to(g, rel).to(torch.float32)


def climate2d(nx: int = 3600, ny: int = 1800, seed: int = 4, rel: float = 1e-3, device="cpu"):
    """f(lon, lat) = 288 - 40 sin^2(lat) + 5 G1 + 0.5 G2, G1 ~ k^-3, G2 ~ k^-1.
    Non-periodic, simply connected domain; shape (1, ny, nx)."""
    g1 = grf((ny, nx), lambda k: k ** -3.0, seed, device)
    g2 = grf((ny, nx), lambda k: k ** -1.0, seed + 1000, device)
    lat = torch.linspace(-math.pi / 2, math.pi / 2, ny, dtype=torch.float64, device=device)
    f = 288.0 - 40.0 * torch.sin(lat)[:, None] ** 2 + 5.0 * g1 + 0.5 * g2
    return _shift_min_to(f, rel).to(torch.float32).reshape(1, ny, nx)


def decompress(f32: torch.Tensor, xi: float, seed: int, mode: str = "uniform") -> torch.Tensor:
    """Simulated error-bounded decompression with |ghat - f| <= xi exactly.

    uniform: ghat = RN_f32(f + xi*u), u ~ counter-based U[-1,1).
    sz:      ghat = RN_f32(2xi * round(f / 2xi)) (SZ-like bins: plateaus/ties).
    Values outside [f-xi, f+xi] after rounding are moved inward one float32
    ulp at a time; the test is exact in float64 (f - xi, f + xi are exact in
    double for float32 operands of comparable magnitude)."""
    xi = float(np.float32(xi))  # the bound the C ABI sees is a float32
    f64 = f32.to(torch.float64)
    flat = f64.reshape(-1)
    if mode == "uniform":
        u = uniform_pm1(flat.numel(), seed, device=f32.device).reshape(f64.shape)
        g64 = f64 + xi * u
    elif mode == "sz":
        g64 = 2 * xi * torch.round(f64 / (2 * xi)) if xi > 0 else f64.clone()
    else:
        raise ValueError(mode)
    g = g64.to(torch.float32)
    lo, hi = f64 - xi, f64 + xi
    # exactness of f - xi / f + xi in double (asserted, not assumed)
    assert bool(((lo + xi) == f64).all()) and bool(((hi - xi) == f64).all())
    for _ in range(4):
        below = g.to(torch.float64) < lo
        above = g.to(torch.float64) > hi
        if not bool(below.any()) and not bool(above.any()):
            break
        g = torch.where(below, torch.nextafter(g, torch.full_like(g, math.inf)), g)
        g = torch.where(above, torch.nextafter(g, torch.full_like(g, -math.inf)), g)
    gd = g.to(torch.float64)
    assert bool(((gd >= lo) & (gd <= hi)).all())
    return g


def lo_monotone(f32: torch.Tensor, xi: float) -> bool:
    """Input diagnostic: is x -> RU(x - xi) strictly increasing
    over the sorted distinct values of f?  If not, lossless clamps can tie and
    ESTUCK becomes possible (amb-17).  Computed in double; harness-only."""
    u = torch.unique(f32.reshape(-1))            # sorted distinct float32
    d = u.to(torch.float64) - xi                  # exact in double (see above)
    r = d.to(torch.float32)
    r = torch.where(r.to(torch.float64) < d, torch.nextafter(r, torch.full_like(r, math.inf)), r)
    return bool((r[1:] > r[:-1]).all()) if r.numel() > 1 else True


CONFIGS = {
    # id: (generator, kwargs, rel, noise seed)
    "C1": dict(name="gaussmix16", gen="gaussmix", kw=dict(n=16, K=8, seed=1), rel=1e-2, seed=101),
    "C2": dict(name="nyx512", gen="nyx_like", kw=dict(shape=(512, 512, 512), seed=2), rel=1e-3,
               seed=102),
    "C3": dict(name="combustion560", gen="combustion", kw=dict(shape=(560, 560, 560), seed=3),
               rel=1e-4, seed=103),
    "C4": dict(name="climate3600x1800", gen="climate2d", kw=dict(nx=3600, ny=1800, seed=4),
               rel=1e-3, seed=104),
    "C5": dict(name="nyx1024", gen="nyx_like", kw=dict(shape=(1024, 1024, 1024), seed=5),
               rel=1e-4, seed=105),
}

_GENS = dict(gaussmix=gaussmix, nyx_like=nyx_like, combustion=combustion, climate2d=climate2d)


class _one_thread:
    """CPU generation pinned to one torch thread: the FFT (MKL) and the
    reductions (mean, std, max) split their work by thread count, so the
    bytes of a CPU-generated field depend on it (C2: different SHA-256 at 1
    and 8 threads).  With one thread the bytes are a function of the seed
    only, which the full-size goldens (tests/golden/fullsize_*.json) need."""

    def __init__(self, device):
        self.on = torch.device(device).type == "cpu"

    def __enter__(self):
        if self.on:
            self.n = torch.get_num_threads()
            torch.set_num_threads(1)

    def __exit__(self, *a):
        if self.on:
            torch.set_num_threads(self.n)


def make(config: str, device="cpu", shape=None, mode: str = "uniform", seed_offset: int = 0,
         xi: float | None = None):
    """(f, ghat, xi) for a config id; `shape` overrides the 3D shape (scaled
    samples with the same recipe).  On the CPU the bytes are host- and
    thread-count-independent (see _one_thread).  seed_offset: an independent
    field of the same recipe (weak scaling: one per rank); xi: the bound to
    decompress with instead of the field's own rel * range (the same xi on
    every rank of a weak-scaling run)."""
    with _one_thread(device):
        return _make(config, device, shape, mode, seed_offset, xi)


def _make(config, device, shape, mode, seed_offset=0, xi=None):
    c = CONFIGS[config]
    kw = dict(c["kw"])
    if seed_offset:
        kw["seed"] = kw["seed"] + 1000 * seed_offset
    if shape is not None:
        if c["gen"] == "gaussmix":
            kw["n"] = shape[0]
        elif c["gen"] == "climate2d":
            kw["ny"], kw["nx"] = shape[-2], shape[-1]
        else:
            kw["shape"] = tuple(shape)
    kw["rel"] = c["rel"]
    f = _GENS[c["gen"]](device=device, **kw)
    if xi is None:
        xi = xi_from_rel(f, c["rel"])
    g = decompress(f, xi, c["seed"] + seed_offset, mode=mode)
    return f.contiguous(), g.contiguous(), xi
