"""GPU parity for NEXT-4 through the C ABI, against the oracle:

* multi-label vertices / edges (§VII-B): gsi_build_graph_ml +
  gsi_query_prepare_ml — signature planes and refined C(u) bitmaps bit-exact against the
  oracle's independent re-implementation of reading A19, and R (count, fingerprint, sorted
  table; isomorphism and homomorphism) equal to oracle.match_ml;
* edge isomorphism (§VII-A): gsi_build_line_graph + gsi_query_prepare_line
  — R_E equal to oracle.match_edges (a direct edge-map backtracker, no line graph) and to the
  brute force on tiny graphs, the Fig. 9 star and the K_n closed forms.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as W
from paper_1906_03420_b200 import gsi

pytestmark = pytest.mark.gpu

if gsi.gsi_device_count() == 0:
    pytest.skip("no CUDA device", allow_module_level=True)


def canon(tab):
    return tab[np.lexsort(tab.T[::-1])] if len(tab) else tab


# ------------------------------------------------------------ multi-label --------------
def test_ml_signatures_and_filter_bit_exact():
    g = W.ml_random_graph(3000, 12000, 300, 8, 5, max_vl=3, max_el=2, seed=21)
    graph = gsi.build_ml(g)
    og = oracle.OracleMLGraph(g)
    planes = oracle.signatures_ml(og)
    assert np.array_equal(gsi.gsi_debug_signatures(graph), planes)
    for s in range(6):
        q = W.ml_walk_query(g, 6, 2100 + s)
        p = gsi.prepare_ml(graph, q)
        for mode, distinct in ((0, False), (2, True)):
            bm, cnt = gsi.gsi_debug_filter_prepared(p, g.n, mode)
            obm, ocnt = oracle.filter_ml(og, planes, oracle.query_signatures_ml(q, distinct=distinct), q)
            assert np.array_equal(bm, obm) and np.array_equal(cnt, ocnt), (s, mode)


@pytest.mark.parametrize("seed", [22, 23])
def test_ml_queries_match_oracle(seed):
    g = W.ml_random_graph(3000, 15000, 300, 6, 4, max_vl=3, max_el=2, seed=seed)
    graph = gsi.build_ml(g)
    og = oracle.OracleMLGraph(g)
    done = 0
    for s in range(12):
        q = W.ml_walk_query(g, 4 + s % 4, 100 * seed + s)
        try:
            cnt, fp, otab = oracle.match_ml(og, q, timeout=5.0)
        except oracle.OracleError:
            continue
        if cnt > 1_000_000:
            continue
        p = gsi.prepare_ml(graph, q)
        r = gsi.gsi_query_run(graph, p, want_table=True)
        assert r.count == cnt and r.fingerprint() == fp, s
        assert np.array_equal(canon(r.table()), otab), s
        assert tuple(q.embedding.tolist()) in {tuple(x) for x in r.table().tolist()}
        assert gsi.gsi_query_run(graph, p, fingerprint=False).count == cnt
        assert gsi.gsi_query_run(graph, p, fingerprint=False, small=False, force_paths=1).count == cnt
        try:
            hc, hfp, _ = oracle.match_ml(og, q, hom=True, table=False, timeout=5.0)
        except oracle.OracleError:
            done += 1
            continue
        rh = gsi.gsi_query_run(graph, p, homomorphism=True)
        assert rh.count == hc and rh.fingerprint() == hfp and hc >= cnt
        done += 1
    assert done >= 6


def test_ml_tiny_vs_brute_force():
    for s in range(40):
        g = W.ml_tiny_graph(3000 + s, nlv=3, nle=2)
        if g.m == 0:
            continue
        q = W.ml_random_query(3100 + s, 2 + s % 3, nlv=3, nle=2)
        graph = gsi.build_ml(g)
        bf = oracle.brute_force_ml(g, q)
        r = gsi.query_ml(graph, q, want_table=True)
        assert [tuple(x) for x in canon(r.table()).tolist()] == bf, s


def test_ml_api_errors():
    g = W.ml_random_graph(500, 2000, 50, 4, 3, seed=24)
    graph = gsi.build_ml(g)
    q = W.ml_walk_query(g, 4, 2400)
    with pytest.raises(gsi.GsiError):   # a multi-label graph needs the multi-label query entry
        gsi.gsi_query_prepare(graph, np.zeros(4, np.int32), q.src, q.dst, np.zeros(len(q.src), np.int32))
    with pytest.raises(gsi.GsiError):   # replication of multi-label graphs is refused
        gsi.gsi_graph_buffers(graph)
    plain = gsi.build(W.cycle_graph(6))
    with pytest.raises(gsi.GsiError):
        gsi.prepare_ml(plain, q)
    with pytest.raises(gsi.GsiError):   # offsets must start at 0
        gsi.gsi_build_graph_ml(3, [1, 1, 2, 3], [0, 0, 0], [0], [1], [0, 1], [0])


# ------------------------------------------------------------ edge isomorphism ---------
def test_line_tiny_vs_brute_force():
    total = 0
    for s in range(60):
        g = W.random_tiny_graph(4000 + s, nlv=2, nle=2)
        if g.m == 0:
            continue
        q = W.random_connected_query(4100 + s, 2 + s % 3, nlv=2, nle=2, extra=0.3)
        graph = gsi.build_line(g)
        bf = oracle.brute_force_edges(g, q)
        r = gsi.query_line(graph, q, want_table=True)
        assert [tuple(x) for x in canon(r.table()).tolist()] == bf, s
        total += len(bf)
    assert total > 100


def test_line_fig9_and_closed_forms():
    g = W.star_graph(3)   # Fig. 9: three edges sharing v0 -> a triangle in the line graph
    graph = gsi.build_line(g)
    assert gsi.query_line(graph, W.star_query(3)).count == 6
    assert gsi.query_line(graph, W.clique_query(3)).count == 6
    for n in (5, 6):
        g = W.complete_graph(n)
        graph = gsi.build_line(g)
        tri = 6 * (math.comb(n, 3) + n * math.comb(n - 1, 3))
        assert gsi.query_line(graph, W.clique_query(3)).count == tri
        assert gsi.query_line(graph, W.star_query(3)).count == tri
    g = W.cycle_graph(9)
    assert gsi.query_line(gsi.build_line(g), W.path_query(4)).count == 18


def test_line_medium_vs_oracle():
    g = W.chung_lu(3000, 9000, 60, nlv=4, nle=4, seed=25)
    graph = gsi.build_line(g)
    og = oracle.OracleGraph(g)
    adj = W._Adj(g)
    done = 0
    for s in range(10):
        q = W.random_walk_query(g, 4 + s % 3, 2500 + s, adj)
        try:
            cnt, fp, otab = oracle.match_edges(og, g, q, timeout=4.0)
        except oracle.OracleError:
            continue
        r = gsi.query_line(graph, q, want_table=True)
        assert r.count == cnt and r.fingerprint() == fp, s
        assert np.array_equal(canon(r.table()), otab), s
        assert gsi.query_line(graph, q, fingerprint=False).count == cnt
        done += 1
    assert done >= 6
    with pytest.raises(gsi.GsiError):   # a plain graph is not a line graph
        gsi.prepare_line(gsi.build(g), W.path_query(3))
