"""Pins of the oracle's classification, steepest paths, labels and extremum
graph (P-3 .. P-6).

Independent references used here:
  * Alexander duality on the link 2-sphere: for every subset L of the 14 link
    vertices, nlc - nuc + 1 = chi(full subcomplex on L) = V_L - E_L + F_L
    (exhaustive over all 2^14 interior masks);
  * the union-find sweep of sublevel sets (textbook merge tree)
    against a Kruskal sweep of the oracle's extremum graph: the ExTreeM
    equivalence theorem says both give the same merge tree, so a
    wrong classification, steepest pointer or label breaks equality;
  * closed forms on monotone fields and the SPEC worked examples.
"""
import itertools
from collections import Counter, defaultdict

import numpy as np
import pytest


def _link(oracle):
    off = [tuple(int(x) for x in r) for r in oracle.offsets()]
    E = [(a, b) for a in range(14) for b in range(a + 1, 14) if oracle.link_adjacent(a, b)]
    Es = set(E)
    T = [t for t in itertools.combinations(range(14), 3)
         if all(p in Es for p in itertools.combinations(t, 2))]
    return off, E, T


def test_alexander_duality_all_masks(oracle):
    _, E, T = _link(oracle)
    full = (1 << 14) - 1
    hist = Counter()
    for m in range(1 << 14):
        nlc = oracle.mask_components(m)
        nuc = oracle.mask_components(full & ~m)
        VL = bin(m).count("1")
        EL = sum(1 for a, b in E if (m >> a) & 1 and (m >> b) & 1)
        FL = sum(1 for t in T if all((m >> k) & 1 for k in t))
        assert nlc - nuc + 1 == VL - EL + FL, (m, nlc, nuc)
        hist[(nlc, nuc)] += 1
    # SURVEY Appendix A histogram (regression pin of the same enumeration)
    assert hist == Counter({(0, 1): 1, (1, 0): 1, (1, 1): 7500, (1, 2): 3629, (2, 1): 3629,
                            (1, 3): 672, (3, 1): 672, (2, 2): 104, (1, 4): 81, (4, 1): 81,
                            (1, 5): 6, (5, 1): 6, (1, 6): 1, (6, 1): 1})


def test_classify_spec_examples(oracle):
    # centre strictly below all neighbours -> minimum
    h = np.full((3, 3), 5.0, np.float32)
    h[1, 1] = 1.0
    nlc, nuc, cls = oracle.classify(h)
    assert cls[4] == oracle.CLS_MIN
    # f = x + y -> interior regular, (0,0) min, (2,2) max (ties by SoS)
    y, x = np.mgrid[0:3, 0:3]
    nlc, nuc, cls = oracle.classify((x + y).astype(np.float32))
    assert cls[4] == oracle.CLS_REGULAR and cls[0] == oracle.CLS_MIN and cls[8] == oracle.CLS_MAX
    assert sorted(np.nonzero(cls)[0].tolist()) == [0, 8]
    # two-low / two-high cross -> both join and split saddle
    cross = np.array([[0, 5, 1], [5, 3, 5], [2, 5, 0]], np.float32)
    nlc, nuc, cls = oracle.classify(cross)
    assert (nlc[4], nuc[4], cls[4]) == (2, 2, oracle.CLS_SADDLE)


def test_monotone_closed_forms(oracle):
    dims = (5, 4, 3)
    V = 60
    f = np.arange(V, dtype=np.float32).reshape(3, 4, 5)
    nlc, nuc, cls = oracle.classify(f)
    assert np.nonzero(cls == oracle.CLS_MIN)[0].tolist() == [0]
    assert np.nonzero(cls == oracle.CLS_MAX)[0].tolist() == [V - 1]
    assert not (cls == oracle.CLS_SADDLE).any()
    ld, lu = oracle.labels(f)
    assert (ld == 0).all() and (lu == V - 1).all()
    ld, lu = oracle.labels(-f)
    assert (ld == V - 1).all() and (lu == 0).all()
    # a constant field is strictly increasing by index under SoS
    ld, lu = oracle.labels(np.ones((3, 4, 5), np.float32))
    assert (ld == 0).all() and (lu == V - 1).all()


def test_steepest_and_labels_brute_force(oracle):
    rs = np.random.default_rng(3)
    for shape in [(4, 5, 6), (1, 7, 9), (1, 1, 12)]:
        h = rs.integers(0, 6, size=shape).astype(np.float32)  # many ties
        dims = tuple(reversed(shape))
        V = h.size
        flat = h.ravel()
        key = lambda v: (flat[v], v)
        up, dn = oracle.steepest(h)
        ld, lu = oracle.labels(h)
        nlc, nuc, cls = oracle.classify(h)
        for v in range(V):
            star = [v] + oracle.neighbors(dims, v)
            assert dn[v] == min(star, key=key) and up[v] == max(star, key=key)
        for v in range(V):
            w, steps = v, 0
            while dn[w] != w:
                assert key(dn[w]) < key(w)
                w = dn[w]
                steps += 1
                assert steps < V
            assert ld[v] == w and cls[w] == oracle.CLS_MIN
            w = v
            while up[w] != w:
                w = up[w]
            assert lu[v] == w and cls[w] == oracle.CLS_MAX


def test_minus_f_duality(oracle):
    rs = np.random.default_rng(5)
    h = rs.permutation(6 * 5 * 4).astype(np.float32).reshape(4, 5, 6)  # tie-free
    a = oracle.classify(h)
    b = oracle.classify(-h)
    assert np.array_equal(a[0], b[1]) and np.array_equal(a[1], b[0])


def test_extremum_graph_spec_examples(oracle):
    f = np.arange(27, dtype=np.float32).reshape(3, 3, 3)
    assert oracle.extremum_graph(f) == set()           # single minimum
    # two basins (minima 5 and 9) separated by one saddle (7); the
    # same saddle splits two maxima (2 and 12, equal values)
    gx = np.array([0, 2, 3, 2, 1], np.float32)
    f = (10 * np.abs(np.arange(3)[:, None] - 1) + gx[None, :]).astype(np.float32)
    assert oracle.extremum_graph(f) == {(7, 5), (7, 9)}
    assert oracle.extremum_graph(f, split=True) == {(7, 2), (7, 12)}
    ref = oracle.reference(f)
    assert ref["S"].tolist() == [7] and ref["J"].tolist() == [7] and ref["P"].tolist() == [7]
    # EGP: the saddle pairs with the higher minimum, f_9 = 1 > f_5 = 0
    assert ref["m1"].tolist() == [9]
    # split: the lower maximum; f_2 == f_12 -> SoS makes 2 the smaller
    assert ref["M1"].tolist() == [2]
    # boundary vertices are real critical points (amb-4): the cross field has
    # boundary join saddles at 1 and 3 besides the centre
    cross = np.array([[0, 5, 1], [5, 3, 5], [2, 5, 0]], np.float32)
    assert oracle.extremum_graph(cross) == {(1, 0), (1, 2), (3, 0), (3, 6), (4, 0), (4, 8)}


def eg_sweep(oracle, h, split):
    """Kruskal sweep of the extremum graph (ExTreeM Step 2 in the elder-rule form)."""
    flat = h.ravel()
    V = flat.size
    sgn = -1 if split else 1
    rank = lambda v: (sgn * flat[v], sgn * v)
    adj = defaultdict(list)
    for s, m in oracle.extremum_graph(h, split=split):
        adj[s].append(m)
    parent, head, birth = {}, {}, {}

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for s in adj:
        for m in adj[s]:
            if m not in parent:
                parent[m], head[m], birth[m] = m, m, m
    arcs, pairs = set(), set()
    for s in sorted(adj, key=rank):
        roots = sorted({find(m) for m in adj[s]}, key=lambda r: rank(birth[r]))
        if len(roots) < 2:
            continue
        for r in roots:
            arcs.add((head[r], s))
            if r != roots[0]:
                pairs.add((birth[r], s))
        parent[s], head[s], birth[s] = s, s, birth[roots[0]]
        for r in roots:
            parent[r] = s
    order = sorted(range(V), key=rank)
    gmin, gmax = order[0], order[-1]
    # the final component: the one containing the global minimum
    if gmin in parent:
        arcs.add((head[find(gmin)], gmax))
    else:
        arcs.add((gmin, gmax))
    pairs.add((gmin, gmax))
    return arcs, pairs


# 1D grids are excluded: with extremum precedence (amb-5) an
# interior 1D maximum is a max, not a join saddle, so the EG has no saddles
# while sublevel components do merge there; the theorem is about 2D/3D.
SHAPES = [(1, 5, 5), (1, 6, 7), (8, 8, 8), (4, 6, 7), (3, 3, 3), (5, 2, 6), (2, 1, 9)]


@pytest.mark.parametrize("shape", SHAPES)
def test_extremum_graph_merge_tree_equivalence(oracle, shape):
    """P:172-173 (ExTreeM): merge tree from the EG == merge tree of the field,
    on random fields up to 8^3, with and without ties."""
    rs = np.random.default_rng(sum(shape))
    n_fields = 30
    for k in range(n_fields):
        if k % 3 == 2:
            h = rs.integers(0, 5, size=shape).astype(np.float32)      # plateaus
        else:
            h = rs.standard_normal(shape).astype(np.float32)
        for split in (False, True):
            arcs, pairs = oracle.merge_tree(h, split=split)
            earcs, epairs = eg_sweep(oracle, h, split)
            assert earcs == arcs, (shape, k, split)
            assert epairs == pairs, (shape, k, split)
            nlc, nuc, cls = oracle.classify(h)
            n_ext = int((cls == (oracle.CLS_MAX if split else oracle.CLS_MIN)).sum())
            assert len(pairs) == n_ext  # one branch per extremum
