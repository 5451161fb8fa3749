"""Pins for the CPU oracle (runs with -m "not gpu").

The oracle is checked against things other than itself (task rule ③):
  * the paper's printed worked example (Fig. 1 / Fig. 7 numbers, tests/golden/fig1.txt);
  * closed forms (K_k in K_n = n!/(n-k)!, P_k in C_n = 2n, C_4 in a grid = 8(a-1)(b-1),
    stars, single edges, bipartite triangles);
  * brute force over every injective map on tiny random graphs (a second, independent
    matcher written straight from Def. 2);
  * invariants of the signature filter (soundness, label exactness, 2-bit group states).
"""
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_golden_fig1():
    """Parse tests/golden/fig1.txt (text graph format of SPEC.md L91-96 plus expectations)."""
    vl, edges, q_vl, q_edges, expect = {}, [], {}, [], {}
    section = None
    for line in open(os.path.join(GOLDEN, "fig1.txt")):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        if tok[0] in ("G", "Q", "EXPECT"):
            section = tok[0]
            continue
        if section == "G":
            if tok[0] == "v":
                vl[int(tok[1])] = int(tok[2])
            elif tok[0] == "e":
                edges.append(tuple(map(int, tok[1:4])))
        elif section == "Q":
            if tok[0] == "v":
                q_vl[int(tok[1])] = int(tok[2])
            elif tok[0] == "e":
                q_edges.append(tuple(map(int, tok[1:4])))
        else:
            expect[tok[0]] = [int(x) for x in tok[1:]]
    n = max(vl) + 1
    g = W.Graph(n, np.array([vl[i] for i in range(n)]), np.array([e[0] for e in edges]),
                np.array([e[1] for e in edges]), np.array([e[2] for e in edges]))
    k = max(q_vl) + 1
    q = W.Query(k, np.array([q_vl[i] for i in range(k)]), np.array([e[0] for e in q_edges]),
                np.array([e[1] for e in q_edges]), np.array([e[2] for e in q_edges]))
    return g, q, expect


# ------------------------------------------------------------------ Fig. 1 / Fig. 7
def test_golden_fixture_matches_generator():
    g, q, _ = load_golden_fig1()
    g2, q2 = W.fig1()
    key = lambda G: sorted(zip(G.src.tolist(), G.dst.tolist(), G.elabels.tolist()))
    assert key(g) == key(g2) and g.vlabels.tolist() == g2.vlabels.tolist()
    assert key(q) == key(q2) and q.vlabels.tolist() == q2.vlabels.tolist()


def test_fig1_printed_values():
    """Every number PAPER.md prints about the running example, computed from the fixture
    with the oracle's N(v,l) (L652, L746-747, L981, L1064-1068, L1089-1091)."""
    g, q, ex = load_golden_fig1()
    og = oracle.OracleGraph(g)
    a, b = 0, 1
    # L746-747: N(v0,a) is the 100-long run v1..v100
    assert og.neighbors(0, a).tolist() == list(range(1, 101))
    # L652: P(G,b) has four vertices {v0,v1,v101,v201} and two edges
    pb = [v for v in range(g.n) if len(og.neighbors(v, b))]
    assert pb == [0, 1, 101, 201] and int((g.elabels == b).sum()) == 2
    # L1064-1066: M = {(v0,vj)}, first edge u1u2 (label a): |GBA| = 200, buf_99 at 197, |buf_99| = 3
    lens = [len(og.neighbors(j, a)) for j in range(1, 101)]
    F = np.concatenate([[0], np.cumsum(lens)])
    assert F[-1] == ex["GBA_u1u2"][0] == 200
    assert F[99] == ex["BUF99_OFFSET"][0] == 197 and lens[99] == ex["BUF99_LEN"][0] == 3
    # L1067: first edge u0u2 (label b) gives |GBA| = 100
    assert sum(len(og.neighbors(0, b)) for _ in range(1, 101)) == ex["GBA_u0u2"][0] == 100
    # L1089-1091: m_99 = (v0, v100): N(v100,a) \ m_99 = {v200, v201}; n C(u2); n N(v0,b) = {v201}
    buf = [x for x in og.neighbors(100, a).tolist() if x not in (0, 100)]
    assert buf == ex["BUF99_AFTER_SUBTRACT"] == [200, 201]
    buf = [x for x in buf if g.vlabels[x] == q.vlabels[2]]          # label-class C(u2) (L576)
    buf = [x for x in buf if x in set(og.neighbors(0, b).tolist())]
    assert buf == ex["BUF99_FINAL"] == [201]


def test_fig1_match_set():
    """The single match of the (draft) result table."""
    g, q, ex = load_golden_fig1()
    og = oracle.OracleGraph(g)
    for root in range(q.n):
        cnt, fp, tab = oracle.match(og, q, root=root)
        assert cnt == 1 and tab.tolist() == [ex["MATCH"]]
        assert fp == oracle.fingerprint_rows(tab, q.n)


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("n,k", [(5, 1), (5, 2), (6, 3), (7, 4), (7, 5), (8, 3)])
def test_clique_in_complete_graph(n, k):
    """Ordered k-cliques of K_n: n!/(n-k)! (non-induced mapping semantics, readings A1/A2)."""
    og = oracle.OracleGraph(W.complete_graph(n))
    cnt, _, tab = oracle.match(og, W.clique_query(k))
    assert cnt == math.perm(n, k) == len({tuple(r) for r in tab.tolist()})


@pytest.mark.parametrize("n,k", [(5, 2), (7, 3), (9, 5), (12, 12), (30, 7)])
def test_path_in_cycle(n, k):
    og = oracle.OracleGraph(W.cycle_graph(n))
    cnt, _, _ = oracle.match(og, W.path_query(k), table=False)
    assert cnt == 2 * n


@pytest.mark.parametrize("a,b", [(2, 2), (3, 4), (5, 7)])
def test_square_in_grid(a, b):
    og = oracle.OracleGraph(W.grid_graph(a, b))
    cnt, _, _ = oracle.match(og, W.cycle_query(4), table=False)
    assert cnt == 8 * (a - 1) * (b - 1)


@pytest.mark.parametrize("leaves", [1, 2, 3])
def test_star_counts(leaves):
    g = W.chung_lu(300, 1200, 40, nlv=1, nle=1, seed=3)
    og = oracle.OracleGraph(g)
    deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=g.n)
    expect = sum(math.perm(int(d), leaves) for d in deg)
    cnt, _, _ = oracle.match(og, W.star_query(leaves), table=False)
    assert cnt == expect


def test_single_edge_is_twice_frequency():
    g = W.chung_lu(500, 3000, 60, nlv=1, nle=5, seed=4)
    og = oracle.OracleGraph(g)
    for l in range(5):
        cnt, _, _ = oracle.match(og, W.edge_query(0, 0, l), table=False)
        assert cnt == 2 * int((g.elabels == l).sum())


def test_triangle_in_bipartite_is_zero():
    pairs = [(i, j) for i in range(5) for j in range(5, 11)]
    g = W.Graph(11, np.zeros(11), np.array([p[0] for p in pairs]), np.array([p[1] for p in pairs]), np.zeros(len(pairs)))
    assert oracle.match(oracle.OracleGraph(g), W.clique_query(3), table=False)[0] == 0
    assert oracle.match(oracle.OracleGraph(g), W.cycle_query(4), table=False)[0] == math.perm(5, 2) * math.perm(6, 2) * 2


def test_per_level_closed_forms():
    """Prefix sub-queries (the per-level tables M_t of a path join order): P_t in C_n = 2n for
    t >= 2 and n for t = 1; K_t in K_n = n!/(n-t)! for every t (SURVEY.md §8(c) 'Per-level M')."""
    og = oracle.OracleGraph(W.cycle_graph(11))
    assert oracle.match(og, W.path_query(1), table=False)[0] == 11
    for t in range(2, 9):
        assert oracle.match(og, W.path_query(t), table=False)[0] == 22
    og = oracle.OracleGraph(W.complete_graph(7))
    for t in range(1, 6):
        assert oracle.match(og, W.clique_query(t), table=False)[0] == math.perm(7, t)


# ------------------------------------------------------------------ brute force
def _tiny_cases(count):
    for s in range(count):
        g = W.random_tiny_graph(s, nlv=1 + s % 3, nle=1 + s % 2)
        k = 1 + s % 5
        q = None
        if s % 2 == 0 and g.m > 0:
            try:
                q = W.random_walk_query(g, k, 10_000 + s, max_restarts=50)
            except ValueError:
                q = None
        if q is None:
            q = W.random_connected_query(10_000 + s, k, nlv=1 + s % 3, nle=1 + s % 2)
        yield s, g, q


def test_backtracker_equals_brute_force():
    """1 000 seeded tiny instances (n <= 9, |L_V| <= 3, |L_E| <= 2, k <= 5): the backtracker's
    sorted table equals the exhaustive enumeration of all injective maps."""
    nonzero = 0
    for s, g, q in _tiny_cases(1000):
        bf = oracle.brute_force(g, q)
        cnt, fp, tab = oracle.match(oracle.OracleGraph(g), q, root=s % q.n)
        assert cnt == len(bf), s
        assert [tuple(r) for r in tab.tolist()] == bf, s
        nonzero += cnt > 0
    assert nonzero > 300


def test_homomorphism_brute_force():
    """Homomorphism = iso without the subtraction; R_hom ⊇ R_iso."""
    for s, g, q in _tiny_cases(120):
        og = oracle.OracleGraph(g)
        bf = oracle.brute_force(g, q, hom=True)
        cnt, _, tab = oracle.match(og, q, hom=True)
        assert [tuple(r) for r in tab.tolist()] == bf, s
        iso = {tuple(r) for r in oracle.match(og, q)[2].tolist()}
        assert iso <= set(bf)


def test_root_restriction_partitions_the_result():
    g = W.chung_lu(400, 2400, 50, nlv=3, nle=3, seed=9)
    og = oracle.OracleGraph(g)
    for qs in range(5):
        q = W.random_walk_query(g, 5, 500 + qs)
        cnt, fp, tab = oracle.match(og, q, root=0)
        parts = np.array_split(np.arange(g.n), 3)
        tot, rows = 0, []
        for p in parts:
            c, _, t = oracle.match(og, q, root=0, roots=p)
            tot += c
            rows += [tuple(r) for r in t.tolist()]
            assert np.isin(t[:, 0], p).all()
        assert tot == cnt and sorted(rows) == [tuple(r) for r in tab.tolist()]
        assert tuple(q.embedding.tolist()) in set(rows)       # the walk's own source embedding


def test_threads_deterministic():
    g = W.chung_lu(2000, 12000, 200, nlv=3, nle=3, seed=11)
    og = oracle.OracleGraph(g)
    q = W.random_walk_query(g, 6, 77)
    a = oracle.match(og, q, threads=1)
    b = oracle.match(og, q, threads=4)
    assert a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2])


def test_errors():
    g = W.cycle_graph(5)
    og = oracle.OracleGraph(g)
    disc = W.Query(4, np.zeros(4), np.array([0, 2]), np.array([1, 3]), np.zeros(2))
    with pytest.raises(oracle.OracleError) as e:
        oracle.match(og, disc)
    assert e.value.code == -6
    bad = W.Graph(3, np.zeros(3), np.array([0, 1]), np.array([0, 2]), np.zeros(2))
    with pytest.raises(oracle.OracleError) as e:
        oracle.OracleGraph(bad)
    assert e.value.code == -4
    dup = W.Graph(3, np.zeros(3), np.array([0, 1]), np.array([1, 0]), np.zeros(2))
    with pytest.raises(oracle.OracleError) as e:
        oracle.OracleGraph(dup)
    assert e.value.code == -5
    par = W.Graph(3, np.zeros(3), np.array([0, 1]), np.array([1, 0]), np.array([0, 1]))
    oracle.OracleGraph(par)                                   # distinct labels: allowed (A3)


# ------------------------------------------------------------------ signatures / filter
def _groups(planes_col):
    """Decode 240 two-bit group states of one signature (planes 1..15)."""
    st = []
    for w in range(1, 16):
        for gi in range(16):
            st.append((int(planes_col[w]) >> (2 * gi)) & 3)
    return st


def test_signature_states_and_label_field():
    g = W.chung_lu(300, 1500, 40, nlv=4, nle=3, seed=5)
    og = oracle.OracleGraph(g)
    planes = oracle.signatures(og)
    assert planes[0].tolist() == g.vlabels.tolist()                  # stored directly (L1277)
    for v in range(g.n):
        st = _groups(planes[:, v])
        assert 2 not in st                                           # states 00/01/11 only (L539)
        # aggregation: state = min(#pairs hashed to the group, 2) (reading A5)
        cnt = np.zeros(240, int)
        for l in range(3):
            for w in og.neighbors(v, l).tolist():
                cnt[oracle.sig_group(l, int(g.vlabels[w]))] += 1
        expect = [0 if c == 0 else (1 if c == 1 else 3) for c in cnt]
        assert st == expect


def test_signature_isolated_and_single_pair():
    g = W.Graph(3, np.array([5, 6, 7]), np.array([0]), np.array([1]), np.array([2]))
    planes = oracle.signatures(oracle.OracleGraph(g))
    assert planes[:, 2].tolist() == [7] + [0] * 15                  # isolated vertex
    st = _groups(planes[:, 0])
    assert sorted(st)[-1] == 1 and sum(st) == 1                      # exactly one 01 group
    assert st.index(1) == oracle.sig_group(2, 6)


def test_filter_sound_and_label_exact():
    """Soundness: every f(u) of every match is in C(u) (S(v)&S(u) = S(u) is necessary,
    PAPER.md L543); label exactness C(u) ⊆ {v : L_V(v) = L_V(u)} (reading A4)."""
    g = W.chung_lu(3000, 15000, 300, nlv=4, nle=6, seed=6)
    og = oracle.OracleGraph(g)
    planes = oracle.signatures(og)
    for s in range(8):
        q = W.random_walk_query(g, 5, 900 + s)
        qsig = oracle.query_signatures(q)
        bm, cnt = oracle.filter(og, planes, qsig)
        bits = np.unpackbits(bm.view(np.uint8), axis=1, bitorder="little")[:, : g.n]
        assert (bits.sum(1) == cnt).all()
        for u in range(q.n):
            assert set(np.nonzero(bits[u])[0]) <= set(np.nonzero(g.vlabels == q.vlabels[u])[0])
        _, _, tab = oracle.match(og, q)
        assert len(tab) > 0
        for u in range(q.n):
            assert bits[u, tab[:, u]].all()


def test_filter_isolated_query_vertex_is_label_class():
    g = W.chung_lu(500, 2000, 50, nlv=3, nle=2, seed=8)
    og = oracle.OracleGraph(g)
    q = W.Query(1, np.array([1]), np.zeros(0), np.zeros(0), np.zeros(0))
    bm, cnt = oracle.filter(og, oracle.signatures(og), oracle.query_signatures(q))
    assert cnt[0] == int((g.vlabels == 1).sum())


def test_fig1_default_filter_sizes():
    """SURVEY.md §8(c) 'C1 default-path trace': with no collision among the 6 keys,
    |C(u)| = (1, 1, 1, 100) and C(u0)={v0}, C(u1)={v100}, C(u2)={v201}."""
    g, q = W.fig1()
    og = oracle.OracleGraph(g)
    bm, cnt = oracle.filter(og, oracle.signatures(og), oracle.query_signatures(q))
    assert cnt.tolist() == [1, 1, 1, 100]
    bits = np.unpackbits(bm.view(np.uint8), axis=1, bitorder="little")[:, : g.n]
    assert np.nonzero(bits[0])[0].tolist() == [0]
    assert np.nonzero(bits[1])[0].tolist() == [100]
    assert np.nonzero(bits[2])[0].tolist() == [201]


def test_homomorphism_filter_sound_with_distinct_keys():
    """Under homomorphism two query neighbours with the same (edge label, neighbour label) key
    may map to one data vertex, so only the distinct-key query encoding is necessary: every
    f(u) of every homomorphic match passes it (reading A5)."""
    for s in range(60):
        g = W.random_tiny_graph(400 + s, nlv=1 + s % 2, nle=1 + s % 2)
        q = W.random_connected_query(40_000 + s, 2 + s % 4, nlv=1 + s % 2, nle=1 + s % 2, extra=0.5)
        og = oracle.OracleGraph(g)
        bm, _ = oracle.filter(og, oracle.signatures(og), oracle.query_signatures(q, distinct=True))
        bits = np.unpackbits(bm.view(np.uint8), axis=1, bitorder="little")[:, : g.n]
        for row in oracle.brute_force(g, q, hom=True):
            for u, v in enumerate(row):
                assert bits[u, v], (s, row)


def test_partial_count_on_timeout():
    """Timed-out count-only runs report the matches found so far (a prefix of the search)."""
    g = W.chung_lu(4000, 30000, 500, nlv=1, nle=1, seed=31)
    og = oracle.OracleGraph(g)
    q = W.path_query(6)
    with pytest.raises(oracle.OracleError):
        oracle.match(og, q, table=False, timeout=1e-3)
    c, fp, _ = oracle.match(og, q, table=False, timeout=1e-3, partial=True)
    assert 0 <= c == fp[0]


def test_murmur_known_answers():
    """External known answers for the hash functions of the written spec (DESIGN.md §3,
    readings A6/A7): SMHasher's published verification values of Appleby's MurmurHash2
    (0x27864C1E) and MurmurHash64A (0x1F0D3804) pin the oracle's general byte-string
    restatements; the oracle's 8-byte signature hash must equal the general one on the key's
    8 little-endian bytes."""
    assert oracle.smhasher_verify(0) == 0x27864C1E
    assert oracle.smhasher_verify(1) == 0x1F0D3804
    rng = np.random.default_rng(11)
    for _ in range(200):
        key = int(rng.integers(0, 1 << 63)) * 2 + int(rng.integers(0, 2))
        seed = int(rng.integers(0, 1 << 32))
        assert oracle.murmur64a_key(key, seed) == oracle.murmur64a(key.to_bytes(8, "little"), seed)
    # and the signature groups the oracle derives from it (reading A6: key = L_E << 32 | L_V)
    for le, lv in [(0, 0), (1, 2), (85, 99), (999, 7)]:
        h = oracle.murmur64a(((le << 32) | lv).to_bytes(8, "little"), 0x9747B28C)
        assert oracle.sig_group(le, lv) == h % 240
