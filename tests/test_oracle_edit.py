"""Pins of the oracle's bound arithmetic and bounded edits (O1, O9; P-8, P-9).

RU/RD are checked against exact rational arithmetic (fractions.Fraction);
the edit sequence of one vertex is re-derived with numpy float32 steps
(xi = 0.5, N = 5 -> steps of 0.1f, then the lossless clamp
f - xi, "If a vertex i requires more than N edits, we store the edit in
a lossless manner as the absolute lower bound, f_i - xi").
"""
from fractions import Fraction

import numpy as np
import pytest


def _nextdown(x):
    return np.nextafter(np.float32(x), np.float32(-np.inf))


def _nextup(x):
    return np.nextafter(np.float32(x), np.float32(np.inf))


def test_directed_rounding_exact(oracle):
    rs = np.random.default_rng(11)
    a = (rs.standard_normal(4000) * 10.0 ** rs.integers(-6, 6, 4000)).astype(np.float32)
    b = np.abs(rs.standard_normal(4000) * 10.0 ** rs.integers(-6, 6, 4000)).astype(np.float32)
    a[:10] = [0, -0.0, 1, 1, 1e-45, -1e-45, 3.0, 2.0, 1.5, 0.1]
    b[:10] = [0, 0, 0, 1, 1e-45, 1e-45, 1.0, 0.5, 0.25, 0.1]
    for x, y in zip(a, b):
        ex_sub = Fraction(float(x)) - Fraction(float(y))
        ru = oracle.ru_sub(x, y)
        assert Fraction(float(ru)) >= ex_sub and Fraction(float(_nextdown(ru))) < ex_sub
        ex_add = Fraction(float(x)) + Fraction(float(y))
        rd = oracle.rd_add(x, y)
        assert Fraction(float(rd)) <= ex_add and Fraction(float(_nextup(rd))) > ex_add


def test_validate(oracle):
    f = np.array([1.0, 2.0, 3.0], np.float32)
    xi = np.float32(0.5)
    assert oracle.validate(f, f, xi) == oracle.OK
    assert oracle.validate(f, f + xi, xi) == oracle.OK          # |diff| == xi is allowed
    assert oracle.validate(f, f - xi, xi) == oracle.OK
    g = (f + xi).copy()
    g[1] = _nextup(g[1])
    assert oracle.validate(f, g, xi) == oracle.EBOUND
    g = f.copy()
    g[0] = np.nan
    assert oracle.validate(f, g, xi) == oracle.EINVAL
    assert oracle.validate(f, f, np.float32(-1)) == oracle.EINVAL
    assert oracle.validate(f, f, xi, N=0) == oracle.EINVAL


def test_step_then_lossless_sequence(oracle):
    """A two-vertex flip that only vertex 0 can repair: every pass marks 0.

    f = [2.0, 2.5], fhat = [2.5, 2.0], xi = 0.5, N = 5.  Vertex 0 steps down by
    Delta = 0.1f until it is <_g vertex 1 (value 2.0, index 1 > 0 so a tie is
    already the f order); if N steps are not enough, edit N+1 is f - xi."""
    f = np.array([2.0, 2.5], np.float32)
    g = np.array([2.5, 2.0], np.float32)
    xi = np.float32(0.5)
    assert np.float32(xi / np.float32(5)) == np.float32(0.1)
    lo = np.float32(1.5)  # f_0 - xi, exactly representable
    seen_lossless = False
    for N in (5, 3, 2, 1, 7):
        delta = np.float32(xi / np.float32(N))
        # expected: numpy float32 arithmetic, independent of the oracle's C code
        x, c, iters = g[0], 0, 0
        while not (x <= g[1]):  # vertex 0 must become <= 2.0 (a tie is f's order)
            x = lo if c >= N else max(np.float32(x - delta), lo)
            c += 1
            iters += 1
        seen_lossless |= (c == N + 1)
        r = oracle.correct(f, g, xi, N)
        assert r.status == oracle.OK
        assert r.iters == iters and r.counts.tolist() == [c, 0], N
        assert r.out[0] == x and r.out[1] == g[1]
        assert r.stats.shape[0] == iters + 1 and (r.stats[:-1, 0] == 1).all()
    # N = 5: 2.5 - 5 x 0.1f rounds to 2.0000002 > 2.0, so edit 6 is lossless
    assert seen_lossless


def test_saturated_vertex_is_not_edited(oracle):
    """A marked vertex already at f - xi stays (O9 'saturated'); when every
    marked vertex is saturated the loop stops with ESTUCK (amb-17)."""
    # lo-collapse: f = [0, -1e-9] with xi = 1 -> RU(f - xi) = -1 for both, so
    # at g = lo the tie is broken by index (0 <_g 1) against f (1 <_f 0)
    f = np.array([0.0, -1e-9], np.float32)
    g = np.array([-1.0, -1.0], np.float32)
    r = oracle.correct(f, g, np.float32(1.0), 5)
    assert r.status == oracle.ESTUCK and r.iters == 0
    assert r.out.tolist() == g.tolist() and r.counts.tolist() == [0, 0]


def test_clean_input_zero_iterations(oracle):
    f = np.linspace(1, 2, 27).astype(np.float32).reshape(3, 3, 3)
    r = oracle.correct(f, f, np.float32(0.1))
    assert r.status == oracle.OK and r.iters == 0 and (r.counts == 0).all()
    assert np.array_equal(r.out.view(np.uint32), f.ravel().view(np.uint32))
    # xi = 0 with g = f is the only valid input and is clean (P-8)
    r = oracle.correct(f, f, np.float32(0.0))
    assert r.status == oracle.OK and r.iters == 0


def test_max_iters(oracle):
    f = np.array([2.0, 2.5], np.float32)
    g = np.array([2.5, 2.0], np.float32)
    r = oracle.correct(f, g, np.float32(0.5), 5, max_iters=2)
    assert r.status == oracle.ESTUCK and r.iters == 2 and r.counts[0] == 2
