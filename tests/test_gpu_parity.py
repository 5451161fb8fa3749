"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

All inputs are seeded synthetic graphs from workloads/ (shapes of SURVEY.md §8(d)); every
expected value comes from oracle/ or from the paper's printed numbers.  Integer work: the bar
is bit-exact equality (sorted match tables, C(u) bitmaps, signature planes, PCSR runs).
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


def canon(tab: np.ndarray) -> np.ndarray:
    if len(tab) == 0:
        return tab.reshape(0, tab.shape[1] if tab.ndim == 2 else 0)
    return tab[np.lexsort(tab.T[::-1])]


def strictly_increasing_in_order(tab: np.ndarray, order) -> bool:
    """Rows emitted in pi-column order must be strictly increasing (order-preserving join)."""
    if len(tab) < 2:
        return True
    t = tab[:, list(order)].astype(np.int64)
    a, b = t[:-1], t[1:]
    # lexicographic a < b
    diff = a != b
    first = np.argmax(diff, axis=1)
    anyd = diff.any(axis=1)
    idx = np.arange(len(a))
    return bool(anyd.all() and (a[idx, first] < b[idx, first]).all())


def bounded_queries(g, og, k, seeds, lo=1, hi=2_000_000, want=None):
    """Random-walk queries whose oracle count is in [lo, hi] (so both sides can materialise
    the table); selection uses only the oracle."""
    out = []
    adj = W._Adj(g)
    for s in seeds:
        q = W.random_walk_query(g, k(s) if callable(k) else k, s, adj)
        try:
            c = oracle.match(og, q, table=False, timeout=5.0)[0]
        except oracle.OracleError:
            continue
        if lo <= c <= hi:
            out.append(q)
        if want and len(out) >= want:
            break
    return out


def run_both(g, q, graph=None, og=None, **kw):
    graph = graph or gsi.build(g)
    og = og or oracle.OracleGraph(g)
    r = gsi.query(graph, q, want_table=True, **kw)
    tab = r.table()
    hom = kw.get("homomorphism", False)
    cnt, fp, otab = oracle.match(og, q, hom=hom)
    return r, tab, cnt, fp, otab


# ------------------------------------------------------------------ paper example ----
def test_fig1_default_path():
    """SURVEY.md §8(c) 'C1 default-path trace' and the single match."""
    g, q = W.fig1()
    r, tab, cnt, fp, otab = run_both(g, q)
    assert r.count == 1 == cnt
    assert tab.tolist() == [[0, 100, 201, 200]]
    assert r.fingerprint() == fp
    s = r.stats()
    assert s["cand"][:4] == [1, 1, 1, 100]
    assert s["order"][:4] == [1, 0, 2, 3]
    assert s["rows"][:4] == [1, 1, 1, 1]
    r2 = gsi.query(gsi.build(g), q, e0_mode=1)
    assert r2.stats()["gba"][1:4] == [3, 1, 3]


def test_fig7_prealloc_numbers():
    """Fig. 7: forced order (u0,u1,u2), label-only filter, paper e0:
    first edge u1u2 gives |GBA| = 200; the planner's own first edge (label b) gives 100."""
    g, q = W.fig1()
    graph = gsi.build(g)
    fo = [0, 1, 2, 3]
    r = gsi.query(graph, q, want_table=True, force_order=fo, filter_mode=1, e0_mode=1,
                  force_first_edge=[-1, -1, 1, -1])
    s = r.stats()
    assert s["rows"][1] == 100                       # M = {(v0, vj)}, 100 rows (L572-576)
    assert s["gba"][2] == 200                        # L1066
    assert s["first_edge"][2] == 1
    assert r.table().tolist() == [[0, 100, 201, 200]]
    r = gsi.query(graph, q, force_order=fo, filter_mode=1, e0_mode=1)
    assert r.stats()["gba"][2] == 100                # L1067 (b is the rarer label, L1068)
    assert r.stats()["first_edge"][2] == 0
    assert r.count == 1


# ------------------------------------------------------------------ PCSR -------------
@pytest.mark.parametrize("gpn", [16, 8, 4, 2])
def test_pcsr_lookup_equals_adjacency(gpn):
    """Every (v,l): GPU N(v,l) equals the oracle's label-filtered adjacency;
    Claim 1 is exercised by small gpn (overflow chains)."""
    g = W.chung_lu(3000, 20000, 400, nlv=3, nle=5, seed=21)
    graph = gsi.build(g, gpn=gpn)
    og = oracle.OracleGraph(g)
    info = graph.info()
    vs = np.repeat(np.arange(g.n), 6)
    ls = np.tile(np.arange(6), g.n)                  # label 5 is absent: empty runs
    lens, reads, nb = gsi.gsi_debug_lookup(graph, vs, ls)
    pos = 0
    for v, l, n_ in zip(vs.tolist(), ls.tolist(), lens.tolist()):
        exp = og.neighbors(v, l)
        assert n_ == len(exp)
        assert nb[pos:pos + n_].tolist() == exp.tolist(), (v, l)
        pos += n_
    assert reads.max() <= info["max_chain"]
    if gpn == 2:
        assert info["max_chain"] > 1 and info["overflow_groups"] > 0
    assert info["n_groups"] == sum(len(np.unique(np.concatenate([g.src[g.elabels == l], g.dst[g.elabels == l]])))
                                   for l in range(5))


def test_pcsr_fig1_partition_b():
    g, _ = W.fig1()
    graph = gsi.build(g)
    lens, _, nb = gsi.gsi_debug_lookup(graph, [0, 1, 101, 201, 5], [1, 1, 1, 1, 1])
    assert lens.tolist() == [1, 1, 1, 1, 0]
    lens, _, nb = gsi.gsi_debug_lookup(graph, [0], [0])
    assert nb.tolist() == list(range(1, 101))       # L746-747


# ------------------------------------------------------------------ signatures/filter -
def test_signature_table_bit_exact():
    g = W.chung_lu(5000, 30000, 600, nlv=5, nle=7, seed=22)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    assert np.array_equal(gsi.gsi_debug_signatures(graph), oracle.signatures(og))


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("size", ["small", "large"])
def test_filter_bitmaps_bit_exact(mode, size):
    """Both filter kernels: warp per word (small graphs) and thread per word (n > ~1.2 M; a
    ragged last word, 8- and 24-vertex queries)."""
    if size == "small":
        g = W.chung_lu(5000, 30000, 600, nlv=5, nle=7, seed=23)
        ks = [8] * 6
    else:
        g = W.chung_lu(1_500_007, 6_000_000, 3000, nlv=40, nle=7, seed=23)
        ks = [8, 24, 12]
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    planes = oracle.signatures(og)
    for s, kq in enumerate(ks):
        q = W.random_walk_query(g, kq, 300 + s)
        bm, cnt = gsi.gsi_debug_filter(graph, q.vlabels, q.src, q.dst, q.elabels, filter_mode=mode)
        if mode in (0, 2):
            obm, ocnt = oracle.filter(og, planes, oracle.query_signatures(q, distinct=mode == 2))
        else:
            iso = W.Query(q.n, q.vlabels, np.zeros(0), np.zeros(0), np.zeros(0))   # label-only = no pairs
            obm, ocnt = oracle.filter(og, planes, oracle.query_signatures(iso))
        assert np.array_equal(bm, obm) and np.array_equal(cnt, ocnt)


# ------------------------------------------------------------------ closed forms -----
@pytest.mark.parametrize("small", [True, False])
@pytest.mark.parametrize("n,k", [(6, 2), (7, 4), (8, 5), (9, 3)])
def test_clique_counts_and_levels(n, k, small):
    graph = gsi.build(W.complete_graph(n))
    r = gsi.query(graph, W.clique_query(k), want_table=True, small=small)
    assert r.stats()["variants"].get("small", 0) == (1 if small else 0)
    assert r.count == math.perm(n, k)
    s = r.stats()
    assert s["rows"][:k] == [math.perm(n, t) for t in range(1, k + 1)]
    assert len({tuple(x) for x in r.table().tolist()}) == r.count


@pytest.mark.parametrize("n,k", [(5, 3), (12, 12), (40, 9)])
def test_path_in_cycle_levels(n, k):
    graph = gsi.build(W.cycle_graph(n))
    r = gsi.query(graph, W.path_query(k))
    assert r.count == 2 * n
    s = r.stats()
    assert s["rows"][0] == n and all(x == 2 * n for x in s["rows"][1:k])


def test_square_in_grid_and_star():
    graph = gsi.build(W.grid_graph(6, 9))
    assert gsi.query(graph, W.cycle_query(4)).count == 8 * 5 * 8
    g = W.chung_lu(300, 1200, 40, nlv=1, nle=1, seed=3)
    deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=g.n)
    graph = gsi.build(g)
    for leaves in (1, 2, 3):
        assert gsi.query(graph, W.star_query(leaves)).count == sum(math.perm(int(d), leaves) for d in deg)


# ------------------------------------------------------------------ random parity ----
@pytest.mark.parametrize("small", [True, False])
def test_tiny_random_vs_oracle(small):
    """Seeded tiny instances (n <= 9, k <= 5, parallel edges with distinct labels included),
    through the one-launch small-query path and the regular per-level path."""
    for s in range(300):
        g = W.random_tiny_graph(s, nlv=1 + s % 3, nle=1 + s % 2)
        if g.m == 0:
            continue
        q = W.random_connected_query(20_000 + s, 1 + s % 5, nlv=1 + s % 3, nle=1 + s % 2)
        r, tab, cnt, fp, otab = run_both(g, q, small=small)
        assert r.count == cnt, s
        assert np.array_equal(canon(tab), otab), s
        assert r.fingerprint() == fp, s


@pytest.mark.parametrize("small", [True, False])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_medium_random_walk_queries(seed, small):
    """Power-law graphs with several tiles of rows and ragged tails; exact sorted tables."""
    g = W.chung_lu(20_000, 120_000, 2_000, nlv=16, nle=8, seed=seed)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    qs = bounded_queries(g, og, lambda s: 4 + s % 6, range(5000 + 100 * seed, 5000 + 100 * seed + 40), want=10)
    assert len(qs) >= 5
    for q in qs:
        r, tab, cnt, fp, otab = run_both(g, q, graph, og, small=small)
        assert r.count == cnt and r.fingerprint() == fp
        assert np.array_equal(canon(tab), otab)
        assert strictly_increasing_in_order(tab, r.stats()["order"][:q.n])
        assert tuple(q.embedding.tolist()) in {tuple(x) for x in tab.tolist()}
        assert gsi.query(graph, q, fingerprint=False, small=small).count == cnt


def test_large_counts_fingerprint():
    """10^7-10^9 matches, count-only on the GPU against the oracle's count and set
    fingerprint (SURVEY.md §8(c) parity at scale)."""
    g = W.chung_lu(4000, 30000, 500, nlv=3, nle=4, seed=31)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    shared, fpk = 0, 0
    for s in (700, 703, 705):
        q = W.random_walk_query(g, 6, s)
        cnt, fp, _ = oracle.match(og, q, table=False)
        for sl in (True, False):   # with and without shared N(v,l0) ∩ C(u) lists
            r = gsi.query(graph, q, shared_lists=sl, small=False)
            assert r.count == cnt and r.fingerprint() == fp, (s, sl)
            shared += r.stats()["n_shared_lists"] if sl else 0
            if sl:
                fpk += r.stats()["variants"].get("final_fp", 0)
            r = gsi.query(graph, q, shared_lists=sl, fingerprint=False, small=False)   # count-only kernels
            assert r.count == cnt, (s, sl)
        assert cnt > 10_000_000 or s == 703
    assert shared > 0 and fpk > 0   # the fingerprinted lean last level (k_final_fp) ran


def test_enron_shaped_config():
    """Config C2 (enron-shaped, 36 692 V / 183 831 E, |L_V|=10, |L_E|=100), 12-vertex walks."""
    g = W.make_config("C2")
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    for j in range(10):
        q = W.random_walk_query(g, 12, 1000 + j)
        r, tab, cnt, fp, otab = run_both(g, q, graph, og)
        assert r.count == cnt and np.array_equal(canon(tab), otab)


# ------------------------------------------------------------------ invariances -------
def test_order_e0_and_filter_invariance():
    g = W.chung_lu(4000, 30000, 500, nlv=8, nle=6, seed=31)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    rng = np.random.default_rng(0)
    for q in bounded_queries(g, og, 6, range(700, 760), hi=500_000, want=6):
        _, _, otab = oracle.match(og, q)
        base = canon(gsi.query(graph, q, want_table=True).table())
        assert np.array_equal(base, otab)
        for trial in range(4):
            # random connected order
            order = [int(rng.integers(q.n))]
            while len(order) < q.n:
                cand = [u for u in range(q.n) if u not in order and any(
                    (a == u and b in order) or (b == u and a in order) for a, b in zip(q.src.tolist(), q.dst.tolist()))]
                order.append(int(rng.choice(cand)))
            for e0 in (0, 1):
                for fm in (0, 1):
                    t = gsi.query(graph, q, want_table=True, force_order=order, e0_mode=e0, filter_mode=fm).table()
                    assert np.array_equal(canon(t), otab)


def test_sharding_concatenates_to_full():
    """M-row sharding run sequentially: shards in rank order == 1-GPU table."""
    g = W.chung_lu(20_000, 150_000, 3_000, nlv=16, nle=8, seed=41)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    for q in bounded_queries(g, og, lambda s: 5 + s % 3, range(900, 960), lo=1000, hi=1_000_000, want=4):
        full = gsi.query(graph, q, want_table=True)
        ft = full.table()
        for W_ in (2, 3, 8):
            for smin in (1, 1 << 30):
                parts = [gsi.query(graph, q, want_table=True, shard_rank=r, shard_count=W_, shard_min_rows=smin)
                         for r in range(W_)]
                cat = np.concatenate([p.table() for p in parts])
                assert np.array_equal(cat, ft)
                assert sum(p.count for p in parts) == full.count
                fps = [p.fingerprint() for p in parts]
                assert sum(f[1] for f in fps) % (1 << 64) == full.fingerprint()[1]


def test_roots_restriction_matches_oracle():
    g = W.chung_lu(10_000, 60_000, 900, nlv=8, nle=6, seed=51)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    rng = np.random.default_rng(1)
    for q in bounded_queries(g, og, 6, range(1100, 1160), hi=2_000_000, want=4):
        r0 = gsi.query(graph, q)
        root = r0.stats()["order"][0]
        roots = rng.choice(g.n, 500, replace=False)
        r = gsi.query(graph, q, want_table=True, roots=roots)
        cnt, fp, otab = oracle.match(og, q, root=root, roots=roots)
        assert r.count == cnt and np.array_equal(canon(r.table()), otab)


def test_homomorphism_matches_oracle():
    for s in range(60):
        g = W.random_tiny_graph(100 + s, nlv=1 + s % 2, nle=1 + s % 2)
        if g.m == 0:
            continue
        q = W.random_connected_query(30_000 + s, 2 + s % 4, nlv=1 + s % 2, nle=1 + s % 2)
        graph = gsi.build(g)
        og = oracle.OracleGraph(g)
        cnt, fp, otab = oracle.match(og, q, hom=True)
        for fm in (0, 1):   # signature filter with the distinct-key query encoding, and label-only
            r = gsi.query(graph, q, want_table=True, homomorphism=True, filter_mode=fm)
            assert r.count == cnt and np.array_equal(canon(r.table()), otab), (s, fm)


def test_k1_and_empty_cases():
    g = W.chung_lu(2000, 8000, 100, nlv=3, nle=2, seed=61)
    graph = gsi.build(g)
    q = W.Query(1, np.array([1]), np.zeros(0), np.zeros(0), np.zeros(0))
    r = gsi.query(graph, q, want_table=True)
    assert r.count == int((g.vlabels == 1).sum())
    assert r.table()[:, 0].tolist() == np.nonzero(g.vlabels == 1)[0].tolist()
    assert r.fingerprint() == oracle.match(oracle.OracleGraph(g), q)[1]
    q = W.edge_query(0, 1, 99)                                  # edge label absent from G
    assert gsi.query(graph, q, want_table=True).count == 0
    q = W.edge_query(0, 77, 0)                                  # vertex label absent
    assert gsi.query(graph, q).count == 0


def test_errors():
    g = W.cycle_graph(6)
    graph = gsi.build(g)
    with pytest.raises(gsi.GsiError) as e:
        gsi.gsi_query(graph, [0, 0, 0, 0], [0, 2], [1, 3], [0, 0])
    assert e.value.status == "GSI_ERR_QUERY_DISCONNECTED"
    with pytest.raises(gsi.GsiError) as e:
        gsi.gsi_query(graph, np.zeros(33), np.arange(32), np.arange(1, 33), np.zeros(32))
    assert e.value.status == "GSI_ERR_QUERY_TOO_LARGE"
    for bad, code in [((3, [0, 0, 0], [0], [0], [0]), "GSI_ERR_SELF_LOOP"),
                      ((3, [0, 0, 0], [0, 1], [1, 0], [0, 0]), "GSI_ERR_DUPLICATE_EDGE"),
                      ((3, [0, 0, 0], [0], [5], [0]), "GSI_ERR_VERTEX_RANGE"),
                      ((3, [0, -1, 0], [0], [1], [0]), "GSI_ERR_LABEL_RANGE")]:
        with pytest.raises(gsi.GsiError) as e:
            gsi.gsi_build_graph(*bad)
        assert e.value.status == code
    gsi.gsi_build_graph(3, [0, 0, 0], [0, 1], [1, 0], [0, 1])   # distinct-label parallel edges: OK
    empty = gsi.gsi_build_graph(4, [0, 0, 0, 0], [], [], [])
    assert gsi.query(empty, W.edge_query()).count == 0


def test_prepared_and_buffers_roundtrip():
    g = W.chung_lu(3000, 15000, 300, nlv=3, nle=3, seed=71)
    graph = gsi.build(g)
    q = W.random_walk_query(g, 6, 1300)
    p = gsi.prepare(graph, q)
    a = gsi.gsi_query_run(graph, p, want_table=True)
    b = gsi.query(graph, q, want_table=True)
    assert np.array_equal(a.table(), b.table())
    # replicate the graph through its buffer descriptors (what the NCCL broadcast does)
    import torch
    descs, meta = gsi.gsi_graph_buffers(graph)
    g2, descs2 = gsi.gsi_graph_alloc_like(meta)
    for (n1, p1, b1), (n2, p2, b2) in zip(descs, descs2):
        assert n1 == n2 and b1 == b2
        gsi.torch_view(p2, b2).copy_(gsi.torch_view(p1, b1))
    torch.cuda.synchronize()
    c = gsi.query(g2, q, want_table=True)
    assert np.array_equal(c.table(), b.table())


def test_chunked_execution_invariance():
    """Depth-first chunking of the GBA slot range (memory bound) changes nothing in R nor in
    the row order (SURVEY.md §7 hard part 3)."""
    g = W.chung_lu(20_000, 150_000, 3_000, nlv=16, nle=8, seed=43)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    for q in bounded_queries(g, og, 6, range(1500, 1560), lo=10_000, hi=300_000, want=3):
        full = gsi.query(graph, q, want_table=True)
        cnt, fp, otab = oracle.match(og, q)
        assert full.count == cnt and np.array_equal(canon(full.table()), otab)
        for cs in (2048, 4096 + 17, 50_000):
            r = gsi.query(graph, q, want_table=True, chunk_slots=cs)
            assert np.array_equal(r.table(), full.table())
            r = gsi.query(graph, q, want_table=True, chunk_slots=cs, shared_lists=False)
            assert np.array_equal(r.table(), full.table())
            assert r.fingerprint() == full.fingerprint()
            c = gsi.query(graph, q, chunk_slots=cs)              # count-only path
            assert c.count == cnt and c.fingerprint() == fp
        assert gsi.query(graph, q, chunk_slots=2048).stats()["n_chunks"] >= 1 or full.stats()["gba"][1] < 2048


def test_timeout_partial_prefix():
    g = W.chung_lu(20_000, 150_000, 3_000, nlv=1, nle=2, seed=44)
    graph = gsi.build(g)
    q = W.random_walk_query(g, 7, 1600)
    r = gsi.query(graph, q, timeout_s=1e-6, partial_on_timeout=True, chunk_slots=2048)
    assert r.stats()["capped"] == 1
    with pytest.raises(gsi.GsiError) as e:
        gsi.query(graph, q, timeout_s=1e-6, chunk_slots=2048)
    assert e.value.status == "GSI_ERR_TIMEOUT"


@pytest.mark.parametrize("kernel", ["lean", "warp", "tile"])
def test_count_ahead_matches_oracle(kernel, monkeypatch):
    """Count-only mode counts the last level from the level before it (|N(v,l0) ∩ C(u)| minus
    the row's own vertices in that run, Alg. 3 lines 9-10) — same count as the oracle and as
    enumerating every match; few vertex labels make the subtraction columns many.  Every
    count-ahead kernel: the lean one (common shape), the generic warp-centric one and the
    slot-tiled k_join."""
    monkeypatch.setenv("GSI_CAHEAD_TILE", "1" if kernel == "tile" else "0")
    monkeypatch.setenv("GSI_CAHEAD_NOLEAN", "1" if kernel != "lean" else "0")
    monkeypatch.setenv("GSI_NEXT_NOLEAN", "1" if kernel != "lean" else "0")   # lean J_NEXT (holes) too
    monkeypatch.setenv("GSI_COUNT_NOLEAN", "1" if kernel != "lean" else "0")  # and the enumerating last level
    seen = 0
    for gs, nlv, nle, k in [(81, 1, 2, 6), (82, 2, 3, 7), (83, 3, 4, 6), (84, 2, 1, 5)]:
        g = W.chung_lu(4000, 30000, 500, nlv=nlv, nle=nle, seed=gs)
        graph = gsi.build(g)
        og = oracle.OracleGraph(g)
        for s in range(3):
            q = W.random_walk_query(g, k, 7000 + 10 * gs + s)
            try:
                cnt = oracle.match(og, q, table=False, timeout=20.0)[0]
            except oracle.OracleError:
                continue
            r = gsi.query(graph, q, fingerprint=False, small=False)
            assert r.count == cnt, (gs, s)
            seen += r.stats()["count_ahead"]
            assert gsi.query(graph, q, fingerprint=False, count_ahead=False, small=False).count == cnt
            assert gsi.query(graph, q, fingerprint=False, force_paths=1).count == cnt
            for W_ in (2, 3):   # sharded at the count-ahead level at the latest
                for pcs in (1, 3):
                    assert sum(gsi.query(graph, q, fingerprint=False, shard_rank=r_, shard_count=W_,
                                         shard_pieces=pcs).count for r_ in range(W_)) == cnt
            assert gsi.query(graph, q, fingerprint=False, chunk_slots=4096).count == cnt
            try:
                hc = oracle.match(og, q, table=False, hom=True, timeout=20.0)[0]
            except oracle.OracleError:
                continue
            assert gsi.query(graph, q, fingerprint=False, homomorphism=True, small=False).count == hc
    assert seen >= 4


def test_bench_scale_root_restricted():
    """Parity at the bench's full size (C5m: R-MAT scale 25, 264 M edges) in the bench's
    launch configuration (count-only: count-ahead, projection, shared runs, probe-ahead;
    and the enumerated fingerprint pass), through the root-restricted protocol of SURVEY.md
    §8(c): both sides restricted to f(pi_1) in S for a sample S of pi_1's label class; the
    sample shrinks until the oracle finishes in seconds."""
    import torch
    g = W.make_config("C5m", device="cuda")
    adj = W._Adj(g, device="cuda")
    qs = [W.random_walk_query(g, 12, 1000 + i, adj) for i in (0, 2, 7, 11, 13)]
    del adj
    torch.cuda.empty_cache()
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    rng = np.random.default_rng(5)
    checked = 0
    for q in qs:
        root = gsi.query(graph, q, fingerprint=False, roots=[int(q.embedding[0])]).stats()["order"][0]
        cls = np.nonzero(g.vlabels == q.vlabels[root])[0]
        for ns in (256, 32, 4):
            # the walk's own start for pi_1 is a root with >= 1 match (its embedding is in R)
            roots = np.unique(np.append(rng.choice(cls, min(ns, len(cls)), replace=False), q.embedding[root]))
            try:
                cnt, fp, _ = oracle.match(og, q, root=root, roots=roots, table=False, timeout=15.0)
            except oracle.OracleError:
                continue
            r = gsi.query(graph, q, roots=roots, fingerprint=False)
            assert cnt >= 1 and r.count == cnt, ns
            r = gsi.query(graph, q, roots=roots)
            assert r.count == cnt and r.fingerprint() == fp
            checked += 1
            break
    assert checked >= 3


def test_query_batch_concurrent():
    """gsi_query_run_batch: concurrent queries (own streams and workspaces) give exactly the
    per-query results, in query order, for every concurrency; errors free the whole batch."""
    g = W.chung_lu(20_000, 120_000, 2_000, nlv=8, nle=6, seed=91)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    qs = bounded_queries(g, og, lambda s: 4 + s % 7, range(9100, 9160), hi=3_000_000, want=10)
    assert len(qs) >= 6
    prepared = [gsi.prepare(graph, q) for q in qs]
    single = [gsi.gsi_query_run(graph, p, want_table=True) for p in prepared]
    for conc in (1, 3, 8):
        rs = gsi.gsi_query_run_batch(graph, prepared, concurrency=conc, want_table=True)
        for a, b in zip(rs, single):
            assert a.count == b.count and a.fingerprint() == b.fingerprint()
            assert np.array_equal(a.table(), b.table())
        rs = gsi.gsi_query_run_batch(graph, prepared, concurrency=conc, fingerprint=False)
        assert [r.count for r in rs] == [b.count for b in single]
    for q, b in zip(qs, single):
        assert b.count == oracle.match(og, q, table=False)[0]
    other = gsi.build(W.cycle_graph(5))
    with pytest.raises(gsi.GsiError):
        gsi.gsi_query_run_batch(other, prepared, concurrency=2)


def test_workspace_trim_and_reuse():
    """The per-device query workspace is reused across queries, grows with demand and can be
    freed at any time (gsi_trim_workspace) without changing any result."""
    g = W.chung_lu(20_000, 120_000, 2_000, nlv=8, nle=6, seed=95)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    qs = bounded_queries(g, og, 7, range(9500, 9540), lo=1000, hi=3_000_000, want=4)
    assert qs
    ref = [oracle.match(og, q, table=False)[0] for q in qs]
    for rep in range(2):
        for q, c in zip(qs, ref):
            assert gsi.query(graph, q, fingerprint=False).count == c
            assert gsi.query(graph, q, fingerprint=False, count_ahead=False).count == c
        gsi.gsi_trim_workspace()
        gsi.gsi_trim_workspace(0)
    assert gsi.query(graph, qs[0], fingerprint=False, mem_budget_bytes=64 << 20).count == ref[0]


def test_small_path_equals_regular_and_aborts_cleanly():
    """The one-launch small-query path (k_small_query) gives the regular path's exact results
    (count, fingerprint, table in the same pi order, per-level |M_t|) on C2-shaped queries; a
    query whose levels outgrow its capacity stops the kernel and falls back to the regular path
    with identical results."""
    g = W.make_config("C2")
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    ran = 0
    for j in range(16):
        q = W.random_walk_query(g, 12, 1000 + j)
        a = gsi.query(graph, q, want_table=True)
        b = gsi.query(graph, q, want_table=True, small=False)
        cnt, fp, otab = oracle.match(og, q)
        assert a.count == b.count == cnt and a.fingerprint() == b.fingerprint() == fp
        assert np.array_equal(a.table(), b.table()) and np.array_equal(canon(a.table()), otab)
        sa, sb = a.stats(), b.stats()
        ran += sa["variants"].get("small", 0) and not sa["small_aborted"]
        if sa["variants"].get("small", 0) and not sa["small_aborted"]:
            assert sa["rows"][:q.n] == sb["rows"][:q.n]
        c = gsi.query(graph, q, fingerprint=False)
        assert c.count == cnt
    assert ran >= 12
    # abort: a dense graph whose levels exceed the kernel's row capacity (2^15)
    g2 = W.chung_lu(3000, 40000, 400, nlv=1, nle=1, seed=5)
    graph2 = gsi.build(g2)
    og2 = oracle.OracleGraph(g2)
    q = W.path_query(4)
    r = gsi.query(graph2, q, fingerprint=True)
    assert r.stats()["small_aborted"] > 0
    cnt, fp, _ = oracle.match(og2, q, table=False)
    assert r.count == cnt and r.fingerprint() == fp


@pytest.mark.parametrize("ab", [1, 1 | 2, 1 | 4, 1 | 8, 1 | 16, 31, 1 | 32, 1 | 64, 1 | 32 | 64, 127])
def test_ablation_engine_same_result(ab):
    """NEXT-3: the paper-style engine (warp per row, Alg. 3/4) with each join technique of
    Tables VI-VIII switched off — CR lookup instead of PCSR, two-step output instead of
    Prealloc-Combine, no write cache, naive set operation — gives the oracle's count and
    fingerprint (same R); likewise without the 4-layer balance (32) or
    the block duplicate removal (64) of NEXT-2."""
    g = W.chung_lu(20_000, 120_000, 2_000, nlv=8, nle=6, seed=97)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    qs = bounded_queries(g, og, lambda s: 4 + s % 5, range(9700, 9760), lo=10, hi=3_000_000, want=6)
    assert len(qs) >= 4
    for q in qs:
        cnt, fp, _ = oracle.match(og, q, table=False)
        r = gsi.query(graph, q, ablation=ab)
        assert r.count == cnt and r.fingerprint() == fp, (ab, r.count, cnt)
        v = r.stats()["variants"]
        assert v.get("ablation", 0) > 0 and v.get("small", 0) == 0
        if ab & 4 and q.n > 2:
            assert v.get("two_step", 0) > 0
        assert gsi.query(graph, q, ablation=ab, fingerprint=False).count == cnt
    with pytest.raises(gsi.GsiError):
        gsi.query(graph, qs[0], ablation=ab, want_table=True)


def test_table_writer_on_shared_runs():
    """Table mode on shared N(v,l0) ∩ C(u) runs (k_surv_scan + k_final_table: the Combine
    offsets in closed form per row, every match written straight into the result) gives the
    oracle's sorted table, in the order-preserving pi order, with and without the fingerprint
    and sharded; the slot-tiled J_TABLE kernel gives the same table."""
    g = W.chung_lu(6000, 40000, 600, nlv=3, nle=6, seed=131)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    qs = bounded_queries(g, og, lambda s: 4 + s % 5, range(13100, 13160), lo=50, hi=300_000, want=5)
    assert len(qs) >= 4
    used = 0
    for q in qs:
        cnt, fp, otab = oracle.match(og, q)
        for fpo in (True, False):
            r = gsi.query(graph, q, want_table=True, fingerprint=fpo, force_paths=1, small=False)
            tab = r.table()
            assert r.count == cnt and np.array_equal(canon(tab), otab)
            if fpo:
                assert r.fingerprint() == fp
            st = r.stats()
            assert strictly_increasing_in_order(tab, st["order"][:q.n])
            used += st["variants"].get("final_table", 0) > 0
        parts = [gsi.query(graph, q, want_table=True, force_paths=1, small=False, shard_rank=r_, shard_count=3,
                           shard_pieces=2).table() for r_ in range(3)]
        assert np.array_equal(canon(np.concatenate(parts)), otab)
    assert used >= 4


def test_table_writer_env_off_same_table(monkeypatch):
    """GSI_TABLE_NOLEAN=1 sends the table level back to the slot-tiled k_join<J_TABLE>: the
    same rows in the same order."""
    g = W.chung_lu(6000, 40000, 600, nlv=3, nle=6, seed=132)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    qs = bounded_queries(g, og, 6, range(13200, 13240), lo=50, hi=300_000, want=3)
    assert qs
    for q in qs:
        a = gsi.query(graph, q, want_table=True, force_paths=1, small=False)
        monkeypatch.setenv("GSI_TABLE_NOLEAN", "1")
        b = gsi.query(graph, q, want_table=True, force_paths=1, small=False)
        monkeypatch.delenv("GSI_TABLE_NOLEAN")
        assert b.stats()["variants"].get("final_table", 0) == 0
        assert np.array_equal(a.table(), b.table()) and a.fingerprint() == b.fingerprint()


@pytest.mark.parametrize("ab", [1, 1 | 4, 1 | 8, 1 | 16, 1 | 64])
def test_ablation_balance_layers_on_hubs(ab, monkeypatch):
    """NEXT-2, the 4-layer balance of the paper-style engine: with small
    thresholds W1 / W2 the hub rows of a power-law graph go to the 8-CTA cluster kernel (row
    staged once, read by the other CTAs through distributed shared memory, in-order compaction
    placed by DSMEM count exchange) and the medium rows to the block kernel; count, fingerprint
    and (two-step) the written rows give the oracle's result, and every layer ran."""
    monkeypatch.setenv("GSI_ABL_W1", "96")
    monkeypatch.setenv("GSI_ABL_W2", "24")
    g = W.chung_lu(20_000, 160_000, 4_000, nlv=4, nle=3, seed=141)
    graph = gsi.build(g)
    og = oracle.OracleGraph(g)
    qs = bounded_queries(g, og, lambda s: 3 + s % 4, range(14100, 14160), lo=100, hi=3_000_000, want=6)
    assert len(qs) >= 4
    layers = np.zeros(3, np.int64)
    for q in qs:
        cnt, fp, _ = oracle.match(og, q, table=False)
        r = gsi.query(graph, q, ablation=ab)
        assert r.count == cnt and r.fingerprint() == fp, (ab, r.count, cnt)
        layers += np.array(r.stats()["abl_layer_rows"], np.int64)
        r2 = gsi.query(graph, q, ablation=ab | 32)   # balance off: the same result
        assert r2.count == cnt and r2.fingerprint() == fp
    assert (layers > 0).all(), layers
