"""Pins for the oracle's NEXT-4 extensions (runs with -m "not gpu"):

* multi-label vertices and edges (§VII-B): ``match_ml`` against a
  pure-Python brute force written straight from the changed definition (L1273-1275), the
  reduction to the single-label definition when every set is a singleton, closed forms, and
  the soundness / exactness of the multi-label filter (hashed labels + refine, L1276-1281);
* edge isomorphism (§VII-A, Fig. 9): ``match_edges`` against an
  edge-map brute force, the Fig. 9 star / line-graph example and closed forms (including
  Whitney's triangle / 3-star pair, which the line-graph transform cannot tell apart).
"""
import math

import numpy as np

import oracle
import workloads as W


def _ml_from_single(g):
    """A single-label graph written as a multi-label one (every set a singleton)."""
    n, m = int(g.n), int(g.m)
    return W.MLGraph(n, np.arange(n + 1), g.vlabels, g.src, g.dst, np.arange(m + 1), g.elabels)


def _uniform_ml_complete(n, vset, eset):
    src = [i for i in range(n) for j in range(i + 1, n)]
    dst = [j for i in range(n) for j in range(i + 1, n)]
    m = len(src)
    return W.MLGraph(n, np.arange(n + 1) * len(vset), np.tile(vset, n), np.array(src), np.array(dst),
                     np.arange(m + 1) * len(eset), np.tile(eset, m))


# ------------------------------------------------------------ multi-label --------------
def test_ml_matches_brute_force_on_tiny_graphs():
    total = 0
    for s in range(300):
        g = W.ml_tiny_graph(s, nlv=3, nle=2)
        q = W.ml_random_query(5000 + s, 2 + s % 3, nlv=3, nle=2)
        og = oracle.OracleMLGraph(g)
        hom = s % 5 == 0
        c, fp, t = oracle.match_ml(og, q, hom=hom)
        bf = oracle.brute_force_ml(g, q, hom=hom)
        assert [tuple(x) for x in t.tolist()] == bf, s
        assert fp == oracle.fingerprint_rows(t, q.n)
        total += c
    assert total > 200   # the instances are not all empty


def test_ml_singletons_reduce_to_single_label_definition():
    """With singleton sets, ⊆ is equality: R equals og_match's on the same graph."""
    for s in range(40):
        g = W.random_tiny_graph(300 + s, nlv=2, nle=2)
        keys = {(min(a, b), max(a, b)) for a, b in zip(g.src.tolist(), g.dst.tolist())}
        if len(keys) != g.m:   # a multi-label edge set needs one edge per pair
            continue
        q = W.random_connected_query(400 + s, 2 + s % 3, nlv=2, nle=2)
        c1, fp1, t1 = oracle.match(oracle.OracleGraph(g), q)
        gm = _ml_from_single(g)
        qm = _ml_from_single(q)
        c2, fp2, t2 = oracle.match_ml(oracle.OracleMLGraph(gm), qm)
        assert c1 == c2 and fp1 == fp2 and np.array_equal(t1, t2)


def test_ml_closed_forms():
    """K_n with every vertex {0,1} and every edge {0,1}: a K_k query labelled {1}/{0} has
    n!/(n-k)! matches (only containment matters); a label outside the sets gives 0; a query
    edge asking for both labels {0,1} still matches every ordered pair."""
    n = 6
    g = _uniform_ml_complete(n, [0, 1], [0, 1])
    og = oracle.OracleMLGraph(g)
    for k in (2, 3, 4):
        q = W.clique_query(k)
        qm = W.MLGraph(k, np.arange(k + 1), np.ones(k, np.int32), q.src, q.dst,
                       np.arange(len(q.src) + 1) * 2, np.tile([0, 1], len(q.src)))
        assert oracle.match_ml(og, qm, table=False)[0] == math.factorial(n) // math.factorial(n - k)
        bad = W.MLGraph(k, np.arange(k + 1), np.full(k, 2, np.int32), q.src, q.dst,
                        np.arange(len(q.src) + 1), np.zeros(len(q.src), np.int32))
        assert oracle.match_ml(og, bad, table=False)[0] == 0


def test_ml_filter_sound_and_label_exact():
    """Refined C(u) contains f(u) for every f in R (soundness) and only vertices whose label
    set contains L_V(u) (the refine step of L1279-1281)."""
    g = W.ml_random_graph(3000, 12000, 300, 6, 4, seed=11)
    og = oracle.OracleMLGraph(g)
    planes = oracle.signatures_ml(og)
    for s in range(6):
        q = W.ml_walk_query(g, 5, 600 + s)
        qsig = oracle.query_signatures_ml(q)
        bm, cnt = oracle.filter_ml(og, planes, qsig, q)
        _, _, tab = oracle.match_ml(og, q, timeout=20.0)
        for u in range(q.n):
            bits = np.unpackbits(bm[u].view(np.uint8), bitorder="little")[:g.n].astype(bool)
            assert cnt[u] == bits.sum()
            assert bits[tab[:, u]].all()
            want = set(q.vset(u))
            for v in np.nonzero(bits)[0][:200]:
                assert want <= set(g.vset(int(v)))
            assert bits[int(q.embedding[u])]
        # a vertex missing one query label is never a candidate
        assert tuple(q.embedding.tolist()) in {tuple(r) for r in tab.tolist()}


def test_ml_walk_embedding_is_a_match():
    g = W.ml_random_graph(2000, 8000, 200, 5, 4, seed=3)
    og = oracle.OracleMLGraph(g)
    for s in range(5):
        q = W.ml_walk_query(g, 6, 900 + s)
        _, _, tab = oracle.match_ml(og, q, timeout=20.0)
        assert tuple(q.embedding.tolist()) in {tuple(r) for r in tab.tolist()}


# ------------------------------------------------------------ edge isomorphism ---------
def test_edges_match_brute_force_on_tiny_graphs():
    total = 0
    for s in range(300):
        g = W.random_tiny_graph(700 + s, nlv=2, nle=2)
        q = W.random_connected_query(800 + s, 2 + s % 3, nlv=2, nle=2, extra=0.3)
        c, fp, t = oracle.match_edges(oracle.OracleGraph(g), g, q)
        bf = oracle.brute_force_edges(g, q)
        assert [tuple(x) for x in t.tolist()] == bf, s
        assert fp == oracle.fingerprint_rows(t, len(q.src))
        total += c
    assert total > 500


def test_edges_fig9_star():
    """Fig. 9: e1 = v0v1, e2 = v0v2, e3 = v0v3 pairwise share v0, so
    their line-graph vertices form a triangle.  Every ordering of the three edges is an edge
    isomorphism of the star onto itself (3! = 6), and so is every map from a triangle query
    (its line graph is a triangle too: Whitney's K3 / K_{1,3} pair)."""
    g = W.star_graph(3)
    og = oracle.OracleGraph(g)
    assert oracle.match_edges(og, g, W.star_query(3), table=False)[0] == 6
    assert oracle.match_edges(og, g, W.clique_query(3), table=False)[0] == 6
    assert oracle.match_edges(og, g, W.path_query(3), table=False)[0] == 6   # 2 edges sharing v0


def test_edges_closed_forms():
    for n in (4, 5, 7):
        g = W.star_graph(n)
        og = oracle.OracleGraph(g)
        assert oracle.match_edges(og, g, W.path_query(3), table=False)[0] == n * (n - 1)
        assert oracle.match_edges(og, g, W.edge_query(), table=False)[0] == n
    for n in (4, 5, 6):
        g = W.complete_graph(n)
        og = oracle.OracleGraph(g)
        tri = 6 * (math.comb(n, 3) + n * math.comb(n - 1, 3))
        assert oracle.match_edges(og, g, W.clique_query(3), table=False)[0] == tri
        assert oracle.match_edges(og, g, W.star_query(3), table=False)[0] == tri
    for n in (5, 8, 11):   # a 3-edge path in C_n: n positions x 2 directions
        g = W.cycle_graph(n)
        assert oracle.match_edges(oracle.OracleGraph(g), g, W.path_query(4), table=False)[0] == 2 * n
