"""Pins of the oracle's mesh and order (P-1, P-2).

The mesh is not stated by the paper (amb-1); the pins are the SPEC's worked
examples, the symmetry invariant and the topology of the
Freudenthal link (a triangulated 2-sphere: 14 - 36 + 24 = 2, every edge on
exactly two triangles) — re-derived here from the 24 Kuhn tetrahedra around
a vertex, a third construction independent of the oracle's pairwise rule.
"""
import itertools

import numpy as np
import pytest


def kuhn_link_edges():
    """Link edges of the origin from the Kuhn subdivision of the 8 incident cubes."""
    edges, tets = set(), 0
    for c in itertools.product((-1, 0), repeat=3):
        for perm in itertools.permutations(range(3)):
            pts = [tuple(c)]
            for ax in perm:
                p = list(pts[-1])
                p[ax] += 1
                pts.append(tuple(p))
            if (0, 0, 0) in pts:
                tets += 1
                others = [p for p in pts if p != (0, 0, 0)]
                for a, b in itertools.combinations(others, 2):
                    edges.add(frozenset((a, b)))
    return edges, tets


def test_neighbors_spec_examples(oracle):
    # S:47-49 (3x3 grid, 2D) and the 3x3x3 centre
    assert oracle.neighbors((3, 3, 1), 4) == [0, 1, 3, 5, 7, 8]
    assert oracle.neighbors((3, 3, 1), 0) == [1, 3, 4]
    assert len(oracle.neighbors((3, 3, 3), 13)) == 14


def test_neighbors_symmetric(oracle):
    dims = (4, 3, 5)
    V = 60
    nb = {v: set(oracle.neighbors(dims, v)) for v in range(V)}
    for v in range(V):
        for u in nb[v]:
            assert v in nb[u]
    # 1D: a path graph
    assert oracle.neighbors((5, 1, 1), 2) == [1, 3]


def test_link_graph_is_triangulated_sphere(oracle):
    off = [tuple(int(x) for x in r) for r in oracle.offsets()]
    assert len(set(off)) == 14 and (0, 0, 0) not in off
    E = {frozenset((off[a], off[b])) for a in range(14) for b in range(a + 1, 14)
         if oracle.link_adjacent(a, b)}
    ref_edges, ntets = kuhn_link_edges()
    assert ntets == 24
    assert E == ref_edges
    assert len(E) == 36
    tris = [t for t in itertools.combinations(off, 3)
            if all(frozenset(p) in E for p in itertools.combinations(t, 2))]
    assert len(tris) == 24
    assert 14 - len(E) + len(tris) == 2  # Euler characteristic of S^2
    for e in E:  # closed surface: every edge on exactly two triangles
        assert sum(1 for t in tris if e <= set(t)) == 2
    deg = {p: sum(1 for e in E if p in e) for p in off}
    for p in off:
        nz = sum(1 for x in p if x != 0)
        assert deg[p] == (4 if nz == 2 else 6)


def test_plane_restriction_is_hexagon(oracle):
    off = [tuple(int(x) for x in r) for r in oracle.offsets()]
    plane = [k for k, p in enumerate(off) if p[2] == 0]
    assert len(plane) == 6
    cyc = [(1, 0, 0), (1, 1, 0), (0, 1, 0), (-1, 0, 0), (-1, -1, 0), (0, -1, 0)]
    idx = {p: k for k, p in enumerate(off)}
    for a, b in zip(cyc, cyc[1:] + cyc[:1]):
        assert oracle.link_adjacent(idx[a], idx[b])
    adj_pairs = sum(1 for a, b in itertools.combinations(plane, 2) if oracle.link_adjacent(a, b))
    assert adj_pairs == 6
    # a line restriction: two isolated points
    line = [idx[(1, 0, 0)], idx[(-1, 0, 0)]]
    assert not oracle.link_adjacent(*line)


def test_sos_examples(oracle):
    # (5.0, 3) < (5.0, 7); (1.0, 9) < (2.0, 0); not (2.0, 0) < (1.0, 9)
    h = np.zeros(10, np.float32)
    h[3] = h[7] = 5.0
    assert oracle.sos_less(h, 3, 7) and not oracle.sos_less(h, 7, 3)
    h[9], h[0] = 1.0, 2.0
    assert oracle.sos_less(h, 9, 0) and not oracle.sos_less(h, 0, 9)
    # -0 == +0 under IEEE compare: the index decides (amb-3)
    z = np.array([0.0, -0.0], np.float32)
    assert oracle.sos_less(z, 0, 1) and not oracle.sos_less(z, 1, 0)


def test_sos_strict_total_order(oracle):
    rs = np.random.default_rng(0)
    h = rs.integers(0, 4, 30).astype(np.float32)  # many ties
    n = len(h)
    L = [[oracle.sos_less(h, u, v) for v in range(n)] for u in range(n)]
    for u in range(n):
        assert not L[u][u]
        for v in range(n):
            if u != v:
                assert L[u][v] != L[v][u]
    order = sorted(range(n), key=lambda i: (h[i], i))
    for a, b in zip(order, order[1:]):
        assert L[a][b]
