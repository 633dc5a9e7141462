"""Pins of the reformulated event constraints (NEXT-1): the order
of ALL critical points of f is preserved by adjacent-pair checks (R7),
replacing the label-based C3 rules R5/R6.

  * SPEC S:298-300 examples: a minimum/saddle pair adjacent in the CP order
    and flipped in g gives one violation; g == f gives none; wherever the
    original C3 fires, R7 finds a flipped CP pair (subsumption).
  * The paper's claim behind the reformulation: with the EG
    preserved, ordering all critical points preserves the EGP pairing -> the
    merge trees' arcs AND elder pairs (branch decomposition) equal f's, also
    the root arcs (which the original formulation may change).
"""
import numpy as np
import pytest
import torch

from synth import fields as S


def test_reform_examples(oracle):
    # two minima (5: value 0, 9: value 1) and a saddle 7 in a 3x5 field; in f
    # the CP order has min 9 < saddle 7; in g push min 9 above the saddle's
    # value while keeping it a minimum.
    gx = np.array([0, 2, 3, 2, 1], np.float32)
    f = (10 * np.abs(np.arange(3)[:, None] - 1) + gx[None, :]).astype(np.float32)
    mark, cnt = oracle.check(f, f, flags=oracle.REFORM)
    assert cnt[0] == 0  # g == f -> empty
    g = f.copy()
    g[1, 4] = 1.9  # minimum 9 still a minimum, now above 1.0 .. but below saddle 3.0
    mark, cnt = oracle.check(f, g, flags=oracle.REFORM)
    assert cnt[5] == 0  # CP order unchanged: no R7 violation
    g[1, 4] = 3.5  # now above the saddle (value 3) but a neighbour (2.0 at x=3) is lower
    mark, cnt = oracle.check(f, g, flags=oracle.REFORM | oracle.NO_C2)
    assert cnt[5] >= 1


def test_reform_subsumes_original_c3(oracle):
    rs = np.random.default_rng(21)
    hits = 0
    for k in range(60):
        shape = [(6, 6, 6), (1, 9, 9), (4, 5, 6)][k % 3]
        f = rs.standard_normal(shape).astype(np.float32) + 5
        g = (f + rs.uniform(-0.3, 0.3, shape)).astype(np.float32)
        _, c_orig = oracle.check(f, g, flags=oracle.NO_C2)
        _, c_ref = oracle.check(f, g, flags=oracle.NO_C2 | oracle.REFORM)
        if c_orig[5] + c_orig[6] > 0:
            hits += 1
            assert c_ref[5] > 0, k
        # the local rules are untouched by the mode
        assert (c_orig[1:4] == c_ref[1:4]).all()
    assert hits > 5


def test_reform_preserves_full_merge_trees(oracle):
    rs = np.random.default_rng(0)
    pair_diff_orig = 0
    for k in range(90):
        shape = [(8, 8, 8), (1, 12, 12), (6, 7, 5)][k % 3]
        f = torch.from_numpy(rs.standard_normal(shape).astype(np.float32))
        f = f - f.min() + 1.0
        xi = S.xi_from_rel(f, [1e-2, 5e-2, 1e-1][k % 3])
        g = S.decompress(f, xi, seed=k)
        fn, gn = f.numpy(), g.numpy()
        r = oracle.correct(fn, gn, xi, 5, flags=oracle.REFORM)
        assert r.status == oracle.OK
        out = r.out.reshape(fn.shape)
        mark, cnt = oracle.check(fn, out, flags=oracle.REFORM)
        assert cnt[0] == 0
        a, b = oracle.classify(fn), oracle.classify(out)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        for split in (False, True):
            assert oracle.extremum_graph(fn, split=split) == oracle.extremum_graph(out, split=split)
            A1, P1 = oracle.merge_tree(fn, split=split)
            A2, P2 = oracle.merge_tree(out, split=split)
            assert A1 == A2 and P1 == P2, (k, split)  # arcs incl. root, and pairings
            ro = oracle.correct(fn, gn, xi, 5)
            pair_diff_orig += oracle.merge_tree(ro.out.reshape(fn.shape), split=split)[1] != P1
    assert pair_diff_orig > 0  # the original formulation does not pin pairings
