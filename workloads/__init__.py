"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no signatures, no PCSR, no join):
it only produces labelled data graphs and query graphs as plain integer arrays.
Both sides of every parity check (``oracle/`` and the CUDA library) receive the same
arrays from here.  Random numbers come from ``torch.Generator`` streams keyed by
(seed, purpose) so the same call on the same device is bit-reproducible.

Graph convention (Def. 1): undirected, vertex labels ``vlabels[n]``,
each undirected edge listed ONCE as (src[i], dst[i], elabels[i]); no self-loops and no
duplicate (v, w, l) triples.  Labels are non-negative int32.

Workload shapes follow SURVEY.md §8(d) (Chung-Lu for enron/gowalla, lattice road graph,
R-MAT for the scale-free config, 80/20 labels, random-walk queries of PAPER.md L1348-1353).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Tuple

import numpy as np
import torch

__all__ = [
    "Graph", "Query", "fig1", "complete_graph", "cycle_graph", "grid_graph", "star_graph",
    "path_query", "clique_query", "cycle_query", "star_query", "edge_query",
    "random_tiny_graph", "random_connected_query", "labels_8020", "labels_zipf",
    "chung_lu", "rmat", "road_grid", "random_walk_query", "random_walk_queries", "CONFIGS",
    "make_config", "MLGraph", "MLQuery", "ml_random_graph", "ml_walk_query", "ml_tiny_graph",
    "ml_random_query",
]


@dataclasses.dataclass
class Graph:
    """Labelled undirected graph as int32 numpy arrays (each edge listed once)."""
    n: int
    vlabels: np.ndarray
    src: np.ndarray
    dst: np.ndarray
    elabels: np.ndarray
    name: str = ""

    @property
    def m(self) -> int:
        return int(self.src.shape[0])

    def __post_init__(self):
        self.vlabels = np.ascontiguousarray(self.vlabels, dtype=np.int32)
        self.src = np.ascontiguousarray(self.src, dtype=np.int32)
        self.dst = np.ascontiguousarray(self.dst, dtype=np.int32)
        self.elabels = np.ascontiguousarray(self.elabels, dtype=np.int32)


@dataclasses.dataclass
class Query(Graph):
    """A query graph Q has the same shape as G (SPEC.md 'the data graph G and query graph Q
    share this shape').  ``embedding`` optionally records the data vertex each query vertex
    was taken from (random-walk queries), i.e. one known member of R(Q, G)."""
    embedding: Optional[np.ndarray] = None

    @property
    def k(self) -> int:
        return self.n


# ----------------------------------------------------------------------------------------
# The paper's running example (Fig. 1 / Fig. 7), reconstructed in SURVEY.md §8(c)
# ----------------------------------------------------------------------------------------
A, B, C = 0, 1, 2          # vertex labels
LA, LB = 0, 1              # edge labels a, b


def fig1() -> Tuple[Graph, Query]:
    """Data graph G and query Q of PAPER.md Fig. 1 (the figure itself is missing; this is the
    reconstruction of SURVEY.md §8(c) 'Fig. 1 reconstruction', consistent with every printed
    value: N(v0,a) = {v1..v100} (L746-747), P(G,b) has 4 vertices / 2 edges (L652),
    |N(v100,a)| = 3 with buf_99 at offset 197 (L1064-1066), |GBA| = 200 / 100 (L1066-1067),
    N(v100,a) minus m_99 = {v200, v201} and the final {v201} (L1089-1091), and the single
    match of the draft table (L349-361))."""
    n = 202
    vl = np.empty(n, np.int32)
    vl[0] = A
    vl[1:101] = B
    vl[101:202] = C
    src, dst, el = [], [], []

    def e(a, b, l):
        src.append(a); dst.append(b); el.append(l)

    for j in range(1, 101):          # v0 - vj, label a
        e(0, j, LA)
    for j in range(2, 100):          # vj - v(100+j), label a
        e(j, 100 + j, LA)
    e(100, 200, LA)
    e(100, 201, LA)
    e(0, 201, LB)                    # label b: v0 - v201, v1 - v101
    e(1, 101, LB)
    g = Graph(n, vl, np.array(src), np.array(dst), np.array(el), name="fig1")
    # Q: u0:A u1:B u2:C u3:C ; u0u1=a, u0u2=b, u1u2=a, u1u3=a
    q = Query(4, np.array([A, B, C, C]), np.array([0, 0, 1, 1]), np.array([1, 2, 2, 3]),
              np.array([LA, LB, LA, LA]), name="fig1-Q")
    return g, q


# ----------------------------------------------------------------------------------------
# Closed-form families (pins of SURVEY.md §8(c) 'Whole match set, closed forms')
# ----------------------------------------------------------------------------------------
def _pairs_graph(n, pairs, vlabel=0, elabel=0, name="") -> Graph:
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    return Graph(n, np.full(n, vlabel, np.int32), pairs[:, 0], pairs[:, 1],
                 np.full(len(pairs), elabel, np.int32), name=name)


def complete_graph(n: int, vlabel=0, elabel=0) -> Graph:
    return _pairs_graph(n, [(i, j) for i in range(n) for j in range(i + 1, n)], vlabel, elabel, f"K{n}")


def cycle_graph(n: int, vlabel=0, elabel=0) -> Graph:
    return _pairs_graph(n, [(i, (i + 1) % n) for i in range(n)], vlabel, elabel, f"C{n}")


def grid_graph(a: int, b: int, vlabel=0, elabel=0) -> Graph:
    pairs = []
    for r in range(a):
        for c in range(b):
            v = r * b + c
            if c + 1 < b:
                pairs.append((v, v + 1))
            if r + 1 < a:
                pairs.append((v, v + b))
    return _pairs_graph(a * b, pairs, vlabel, elabel, f"grid{a}x{b}")


def star_graph(leaves: int, vlabel=0, elabel=0) -> Graph:
    return _pairs_graph(leaves + 1, [(0, i) for i in range(1, leaves + 1)], vlabel, elabel, f"star{leaves}")


def _q(k, pairs, vlabel=0, elabel=0, name="") -> Query:
    g = _pairs_graph(k, pairs, vlabel, elabel, name)
    return Query(g.n, g.vlabels, g.src, g.dst, g.elabels, name=name)


def path_query(k: int, vlabel=0, elabel=0) -> Query:
    return _q(k, [(i, i + 1) for i in range(k - 1)], vlabel, elabel, f"P{k}")


def clique_query(k: int, vlabel=0, elabel=0) -> Query:
    return _q(k, [(i, j) for i in range(k) for j in range(i + 1, k)], vlabel, elabel, f"K{k}")


def cycle_query(k: int, vlabel=0, elabel=0) -> Query:
    return _q(k, [(i, (i + 1) % k) for i in range(k)], vlabel, elabel, f"C{k}")


def star_query(leaves: int, vlabel=0, elabel=0) -> Query:
    return _q(leaves + 1, [(0, i) for i in range(1, leaves + 1)], vlabel, elabel, f"S{leaves}")


def edge_query(vlabel_a=0, vlabel_b=0, elabel=0) -> Query:
    return Query(2, np.array([vlabel_a, vlabel_b]), np.array([0]), np.array([1]), np.array([elabel]), name="edge")


# ----------------------------------------------------------------------------------------
# Random generators (torch streams keyed by (seed, purpose))
# ----------------------------------------------------------------------------------------
_PURPOSE = {"topology": 1, "vlabel": 2, "elabel": 3, "perm": 4, "query": 5, "extra": 6, "tiny": 7}


def _gen(seed: int, purpose: str, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + _PURPOSE[purpose] * 7919) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


def labels_8020(count: int, nlabels: int, seed: int, purpose="vlabel", device="cpu") -> torch.Tensor:
    """80/20 label rule (SURVEY.md reading A15; draft PAPER.md L1371-1372): the top
    ceil(0.2 L) labels share 80 % of the mass uniformly, the rest share 20 % uniformly."""
    if nlabels <= 1:
        return torch.zeros(count, dtype=torch.int32, device=device)
    top = max(1, math.ceil(0.2 * nlabels))
    p = torch.empty(nlabels, dtype=torch.float64)
    if top == nlabels:
        p[:] = 1.0 / nlabels
    else:
        p[:top] = 0.8 / top
        p[top:] = 0.2 / (nlabels - top)
    cdf = torch.cumsum(p, 0).to(device)
    cdf[-1] = 1.0
    r = torch.rand(count, generator=_gen(seed, purpose, device), dtype=torch.float64, device=device)
    return torch.searchsorted(cdf, r, right=True).clamp_(max=nlabels - 1).to(torch.int32)


def labels_zipf(count: int, nlabels: int, seed: int, s=1.0, purpose="vlabel", device="cpu") -> torch.Tensor:
    p = 1.0 / torch.arange(1, nlabels + 1, dtype=torch.float64) ** s
    cdf = torch.cumsum(p / p.sum(), 0).to(device)
    cdf[-1] = 1.0
    r = torch.rand(count, generator=_gen(seed, purpose, device), dtype=torch.float64, device=device)
    return torch.searchsorted(cdf, r, right=True).clamp_(max=nlabels - 1).to(torch.int32)


def _canon_unique(u: torch.Tensor, v: torch.Tensor, n: int) -> torch.Tensor:
    """Drop self-loops, canonicalise (min,max) and deduplicate; returns sorted int64 keys."""
    keep = u != v
    u, v = u[keep], v[keep]
    a = torch.minimum(u, v).to(torch.int64)
    b = torch.maximum(u, v).to(torch.int64)
    return torch.unique(a * n + b)


def _finish(n, keys, nlv, nle, seed, name, device, vlabel_fn=labels_8020) -> Graph:
    src = (keys // n).to(torch.int32)
    dst = (keys % n).to(torch.int32)
    vl = vlabel_fn(n, nlv, seed, purpose="vlabel", device=device)
    el = vlabel_fn(src.numel(), nle, seed, purpose="elabel", device=device)
    return Graph(n, vl.cpu().numpy(), src.cpu().numpy(), dst.cpu().numpy(), el.cpu().numpy(), name=name)


def random_tiny_graph(seed: int, n: Optional[int] = None, nlv: int = 2, nle: int = 2, p: float = 0.45) -> Graph:
    """Tiny random graph for brute-force pins (n <= 9, few labels), Erdos-Renyi G(n,p).
    With probability 1/4 one pair gets a second, distinct-label parallel edge."""
    g = _gen(seed, "tiny")
    if n is None:
        n = int(torch.randint(3, 10, (1,), generator=g))
    src, dst, el = [], [], []
    for i in range(n):
        for j in range(i + 1, n):
            if float(torch.rand(1, generator=g)) < p:
                l = int(torch.randint(0, nle, (1,), generator=g))
                src.append(i); dst.append(j); el.append(l)
                if nle > 1 and float(torch.rand(1, generator=g)) < 0.08:
                    src.append(i); dst.append(j); el.append((l + 1) % nle)
    vl = torch.randint(0, nlv, (n,), generator=g).numpy()
    return Graph(n, vl, np.array(src, np.int32), np.array(dst, np.int32), np.array(el, np.int32), name=f"tiny{seed}")


def random_connected_query(seed: int, k: int, nlv: int = 2, nle: int = 2, extra: float = 0.3) -> Query:
    """Random connected query: random spanning tree plus extra edges (labels uniform)."""
    g = _gen(seed, "query")
    src, dst, el = [], [], []
    pairs = set()
    for i in range(1, k):
        j = int(torch.randint(0, i, (1,), generator=g))
        src.append(j); dst.append(i); el.append(int(torch.randint(0, nle, (1,), generator=g)))
        pairs.add((j, i))
    for i in range(k):
        for j in range(i + 1, k):
            if (i, j) not in pairs and float(torch.rand(1, generator=g)) < extra:
                src.append(i); dst.append(j); el.append(int(torch.randint(0, nle, (1,), generator=g)))
    vl = torch.randint(0, nlv, (k,), generator=g).numpy()
    return Query(k, vl, np.array(src, np.int32), np.array(dst, np.int32), np.array(el, np.int32), name=f"rq{seed}")


def chung_lu(n: int, m: int, dmax: float, nlv: int, nle: int, seed: int = 1, device="cpu", name="chung_lu") -> Graph:
    """Chung-Lu power-law graph with exactly m unique undirected edges:
    w_i = c (i+1)^-alpha with alpha bisected so max w = dmax and sum w = 2m; endpoints drawn
    proportional to w; self-loops/duplicates dropped and topped up; ids randomly permuted."""
    i = torch.arange(1, n + 1, dtype=torch.float64)
    target = 2.0 * m / dmax                         # sum (i+1)^-alpha must equal this
    lo, hi = 0.0, 4.0
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        s = float(torch.sum(i ** -mid))
        if s > target:
            lo = mid
        else:
            hi = mid
    alpha = 0.5 * (lo + hi)
    w = i ** -alpha
    cdf = torch.cumsum(w / w.sum(), 0).to(device)
    cdf[-1] = 1.0
    gt = _gen(seed, "topology", device)
    perm = torch.randperm(n, generator=_gen(seed, "perm", device), device=device)
    keys = torch.empty(0, dtype=torch.int64, device=device)
    while keys.numel() < m:
        need = m - keys.numel()
        draw = int(need * 1.3) + 1024
        r1 = torch.rand(draw, generator=gt, dtype=torch.float64, device=device)
        r2 = torch.rand(draw, generator=gt, dtype=torch.float64, device=device)
        u = perm[torch.searchsorted(cdf, r1).clamp_(max=n - 1)]
        v = perm[torch.searchsorted(cdf, r2).clamp_(max=n - 1)]
        new = _canon_unique(u, v, n)
        merged = torch.unique(torch.cat([keys, new]))
        if merged.numel() > m:
            # keep the old keys, add a deterministic subset of the new ones
            fresh = new[~torch.isin(new, keys)]
            fresh = fresh[torch.randperm(fresh.numel(), generator=gt, device=device)[: m - keys.numel()]]
            merged = torch.sort(torch.cat([keys, fresh])).values
        keys = merged
    return _finish(n, keys, nlv, nle, seed, name, device)


def rmat(scale: int, edge_factor: int, nlv: int, nle: int, seed: int = 1,
         abcd=(0.57, 0.19, 0.19, 0.05), device="cpu", name="rmat") -> Graph:
    """R-MAT (Graph500 recipe): 2^scale vertices, edge_factor*2^scale
    samples, quadrant probabilities abcd, seeded random vertex permutation, dedup,
    self-loops removed.  The exact |E| is whatever survives dedup."""
    n = 1 << scale
    ne = edge_factor * n
    a, b, c, _ = abcd
    gt = _gen(seed, "topology", device)
    src = torch.zeros(ne, dtype=torch.int64, device=device)
    dst = torch.zeros(ne, dtype=torch.int64, device=device)
    for lvl in range(scale):
        r = torch.rand(ne, generator=gt, dtype=torch.float32, device=device)
        bs = r >= (a + b)
        bd = ((r >= a) & (r < a + b)) | (r >= (a + b + c))
        src |= bs.to(torch.int64) << lvl
        dst |= bd.to(torch.int64) << lvl
        del r, bs, bd
    perm = torch.randperm(n, generator=_gen(seed, "perm", device), device=device)
    src = perm[src]
    dst = perm[dst]
    keys = _canon_unique(src, dst, n)
    del src, dst
    return _finish(n, keys, nlv, nle, seed, name, device)


def road_grid(side: int, m: int, nlv: int, nle: int, seed: int = 1, device="cpu", name="road") -> Graph:
    """Road-shaped low-degree graph: side x side lattice with row-major
    ids; a random spanning tree (Boruvka over random edge weights) plus uniformly chosen unused
    lattice/diagonal edges until m edges; max degree <= 8."""
    n = side * side
    idx = torch.arange(n, device=device, dtype=torch.int64)
    r, c = idx // side, idx % side
    cand = []
    for dr, dc in ((0, 1), (1, 0), (1, 1), (1, -1)):
        ok = (r + dr < side) & (c + dc >= 0) & (c + dc < side)
        u = idx[ok]
        cand.append(torch.stack([u, u + dr * side + dc], 1))
    lattice = torch.cat(cand[:2])          # axis-aligned edges form the spanning-tree pool
    diag = torch.cat(cand[2:])
    gt = _gen(seed, "topology", device)
    w = torch.randperm(lattice.shape[0], generator=gt, device=device)
    eu, ev = lattice[:, 0], lattice[:, 1]
    comp = idx.clone()
    in_tree = torch.zeros(lattice.shape[0], dtype=torch.bool, device=device)
    big = torch.iinfo(torch.int64).max
    while True:
        cu, cv = comp[eu], comp[ev]
        inter = cu != cv
        if not bool(inter.any()):
            break
        best = torch.full((n,), big, dtype=torch.int64, device=device)
        best.scatter_reduce_(0, cu[inter], w[inter], reduce="amin")
        best.scatter_reduce_(0, cv[inter], w[inter], reduce="amin")
        chosen = inter & ((w == best[cu]) | (w == best[cv]))
        in_tree |= chosen
        # hook: each component points at the other end of its min edge; break 2-cycles
        ptr = idx.clone()
        ce = chosen.nonzero().squeeze(1)
        a_, b_ = cu[ce], cv[ce]
        wa = w[ce]
        sel_a = best[a_] == wa
        ptr[a_[sel_a]] = b_[sel_a]
        sel_b = best[b_] == wa
        ptr[b_[sel_b]] = a_[sel_b]
        mutual = ptr[ptr] == idx
        ptr = torch.where(mutual & (idx < ptr), idx, ptr)
        while True:
            nxt = ptr[ptr]
            if bool((nxt == ptr).all()):
                break
            ptr = nxt
        comp = ptr[comp]
    tree = lattice[in_tree]
    rest = torch.cat([lattice[~in_tree], diag])
    need = max(0, m - tree.shape[0])
    pick = torch.randperm(rest.shape[0], generator=_gen(seed, "extra", device), device=device)[:need]
    edges = torch.cat([tree, rest[pick]])
    keys = torch.sort(edges.min(1).values * n + edges.max(1).values).values
    return _finish(n, keys, nlv, nle, seed, name, device)


# ----------------------------------------------------------------------------------------
# Random-walk queries (SURVEY.md reading A14)
# ----------------------------------------------------------------------------------------
class _Adj:
    """Label-carrying adjacency (CSR over directed entries) used only to walk the graph."""

    def __init__(self, g: Graph, device="cpu"):
        src = torch.as_tensor(g.src, device=device).to(torch.int64)
        dst = torch.as_tensor(g.dst, device=device).to(torch.int64)
        el = torch.as_tensor(g.elabels, device=device)
        s2 = torch.cat([src, dst])
        d2 = torch.cat([dst, src])
        l2 = torch.cat([el, el])
        order = torch.argsort(s2, stable=True)
        self.nbr = d2[order].to(torch.int32).cpu().numpy()
        self.lab = l2[order].cpu().numpy()
        deg = torch.bincount(s2, minlength=g.n)
        del order, s2, d2, l2
        self.off = np.concatenate([[0], torch.cumsum(deg, 0).cpu().numpy()])
        self.deg = deg.cpu().numpy()
        self.nonisolated = np.nonzero(self.deg)[0]


def random_walk_query(g: Graph, k: int, seed: int, adj: Optional[_Adj] = None,
                      max_restarts: int = 1000) -> Query:
    """Walk from a uniformly random non-isolated vertex, each step along a uniformly chosen
    incident edge, until k distinct vertices are visited; Q = the visited vertices and the
    walked edges with their labels (A14: walked edges only; restart after 100k steps without
    a new vertex).  Query ids are first-visit order; ``embedding`` is the source match."""
    adj = adj or _Adj(g)
    rng = np.random.default_rng([seed, _PURPOSE["query"]])
    if len(adj.nonisolated) == 0:
        raise ValueError("graph has no edges")
    for _attempt in range(max_restarts):
        v = int(adj.nonisolated[rng.integers(len(adj.nonisolated))])
        order = {v: 0}
        edges = {}
        stale = 0
        while len(order) < k and stale < 100 * k:
            d = int(adj.deg[v])
            j = int(adj.off[v] + rng.integers(d))
            w, l = int(adj.nbr[j]), int(adj.lab[j])
            new = w not in order
            if new:
                order[w] = len(order)
                stale = 0
            else:
                stale += 1
            a, b = order[v], order[w]
            edges[(min(a, b), max(a, b), l)] = True
            v = w
        if len(order) == k:
            break
    else:
        raise ValueError(f"no connected {k}-vertex walk found after {max_restarts} restarts")
    emb = np.empty(k, np.int64)
    for dv, qi in order.items():
        emb[qi] = dv
    e = np.array(sorted(edges.keys()), dtype=np.int64).reshape(-1, 3)
    return Query(k, g.vlabels[emb], e[:, 0], e[:, 1], e[:, 2], name=f"walk{seed}",
                 embedding=emb.astype(np.int32))


def random_walk_queries(g: Graph, k: int, seeds) -> List[Query]:
    adj = _Adj(g)
    return [random_walk_query(g, k, s, adj) for s in seeds]


# ----------------------------------------------------------------------------------------
# Named configs (BASELINE.json configs)
# ----------------------------------------------------------------------------------------
CONFIGS = {
    # name: (generator, kwargs)
    "C1": ("fig1", {}),
    "C2": ("chung_lu", dict(n=36_692, m=183_831, dmax=1_700, nlv=10, nle=100)),
    "C3": ("chung_lu", dict(n=196_591, m=950_327, dmax=29_000, nlv=100, nle=100)),
    "C4": ("road_grid", dict(side=3_742, m=17_000_000, nlv=1_000, nle=1_000)),
    "C5a": ("rmat", dict(scale=25, edge_factor=8, nlv=1_000, nle=86)),
    "C5b": ("rmat", dict(scale=25, edge_factor=8, nlv=10, nle=86)),
    # join-stress variant sized for a bounded bench: |L_V| = 10 gives 10^10-10^11 matches per
    # 12-vertex walk query at scale 25, |L_V| = 1000 gives 1-100
    "C5m": ("rmat", dict(scale=25, edge_factor=8, nlv=100, nle=86)),
}


def make_config(name: str, seed: int = 1, device="cpu", **override) -> Graph:
    kind, kw = CONFIGS[name]
    kw = dict(kw, **override)
    if kind == "fig1":
        return fig1()[0]
    fn = {"chung_lu": chung_lu, "rmat": rmat, "road_grid": road_grid}[kind]
    return fn(seed=seed, device=device, name=name, **kw)


# ----------------------------------------------------------------------------------------
# Multi-label graphs (§VII-B): vertex label SETS and edge label SETS
# ----------------------------------------------------------------------------------------
_PURPOSE.update({"mlv": 11, "mle": 12, "mlq": 13})


@dataclasses.dataclass
class MLGraph:
    """Undirected graph whose vertices and edges carry label SETS: L_V(v) =
    vls[vls_off[v]:vls_off[v+1]], L_E(e) = els[els_off[e]:els_off[e+1]] (each edge listed once,
    no two edges on the same vertex pair, no self-loops; labels >= 0, no repeats in a set)."""
    n: int
    vls_off: np.ndarray
    vls: np.ndarray
    src: np.ndarray
    dst: np.ndarray
    els_off: np.ndarray
    els: np.ndarray
    name: str = ""
    embedding: Optional[np.ndarray] = None   # queries: the data vertex of each query vertex

    @property
    def m(self) -> int:
        return int(self.src.shape[0])

    def __post_init__(self):
        self.vls_off = np.ascontiguousarray(self.vls_off, dtype=np.int64)
        self.vls = np.ascontiguousarray(self.vls, dtype=np.int32)
        self.src = np.ascontiguousarray(self.src, dtype=np.int32)
        self.dst = np.ascontiguousarray(self.dst, dtype=np.int32)
        self.els_off = np.ascontiguousarray(self.els_off, dtype=np.int64)
        self.els = np.ascontiguousarray(self.els, dtype=np.int32)

    def vset(self, v: int) -> List[int]:
        return self.vls[self.vls_off[v]:self.vls_off[v + 1]].tolist()

    def eset(self, e: int) -> List[int]:
        return self.els[self.els_off[e]:self.els_off[e + 1]].tolist()


MLQuery = MLGraph


def _label_sets(count: int, nlabels: int, max_per: int, seed: int, purpose: str) -> Tuple[np.ndarray, np.ndarray]:
    """1..max_per distinct labels per item, each drawn by the 80/20 rule (reading A15)."""
    g = np.random.default_rng([seed, _PURPOSE[purpose]])
    sizes = g.integers(1, max_per + 1, count)
    draws = labels_8020(int(sizes.sum()), nlabels, seed, purpose=purpose).numpy()
    off = np.zeros(count + 1, np.int64)
    out = []
    pos = 0
    for i in range(count):
        st = sorted(set(draws[pos:pos + sizes[i]].tolist()))
        pos += sizes[i]
        out.extend(st)
        off[i + 1] = len(out)
    return off, np.array(out, np.int32)


def ml_random_graph(n: int, m: int, dmax: float, nlv: int, nle: int, max_vl: int = 3, max_el: int = 2,
                    seed: int = 1, name: str = "ml") -> MLGraph:
    """Chung-Lu topology (as chung_lu) with 1..max_vl vertex labels and 1..max_el edge labels."""
    base = chung_lu(n, m, dmax, 1, 1, seed=seed, name=name)
    voff, vls = _label_sets(n, nlv, max_vl, seed, "mlv")
    eoff, els = _label_sets(base.m, nle, max_el, seed, "mle")
    return MLGraph(n, voff, vls, base.src, base.dst, eoff, els, name=name)


def ml_tiny_graph(seed: int, nlv: int = 3, nle: int = 2) -> MLGraph:
    """Tiny multi-label graph for brute force (n <= 8)."""
    t = random_tiny_graph(seed, nlv=1, nle=1, p=0.5)
    keys = sorted({(min(a, b), max(a, b)) for a, b in zip(t.src.tolist(), t.dst.tolist())})
    src = np.array([a for a, _ in keys], np.int32)
    dst = np.array([b for _, b in keys], np.int32)
    voff, vls = _label_sets(t.n, nlv, 2, seed, "mlv")
    eoff, els = _label_sets(len(keys), nle, 2, seed, "mle")
    return MLGraph(t.n, voff, vls, src, dst, eoff, els, name=f"mltiny{seed}")


def ml_walk_query(g: MLGraph, k: int, seed: int) -> MLGraph:
    """Random-walk query (A14) on a multi-label graph: the walked vertices and edges, each
    query label set a random non-empty subset of its data vertex's / edge's set, so the walk's
    own embedding is a match."""
    plain = Graph(g.n, np.zeros(g.n, np.int32), g.src, g.dst, np.arange(g.m, dtype=np.int32) % (1 << 30))
    q = random_walk_query(plain, k, seed)   # elabels = data edge ids (placeholder labels)
    rng = np.random.default_rng([seed, _PURPOSE["mlq"]])
    emb = q.embedding.astype(np.int64)
    qv_off = np.zeros(k + 1, np.int64)
    qv = []
    for u in range(k):
        st = g.vset(int(emb[u]))
        keep = [x for x in st if rng.random() < 0.6] or [st[int(rng.integers(len(st)))]]
        qv.extend(keep)
        qv_off[u + 1] = len(qv)
    qe_off = np.zeros(len(q.src) + 1, np.int64)
    qe = []
    for i, eid in enumerate(q.elabels.tolist()):
        st = g.eset(int(eid))
        keep = [x for x in st if rng.random() < 0.6] or [st[int(rng.integers(len(st)))]]
        qe.extend(keep)
        qe_off[i + 1] = len(qe)
    return MLGraph(k, qv_off, np.array(qv, np.int32), q.src, q.dst, qe_off, np.array(qe, np.int32),
                   name=f"mlwalk{seed}", embedding=q.embedding)


def ml_random_query(seed: int, k: int, nlv: int = 3, nle: int = 2) -> MLGraph:
    """Random connected multi-label query (spanning tree + extra edges, 1-2 labels each)."""
    q = random_connected_query(seed, k, nlv=1, nle=1, extra=0.3)
    voff, vls = _label_sets(k, nlv, 2, seed + 7, "mlv")
    eoff, els = _label_sets(len(q.src), nle, 2, seed + 7, "mle")
    return MLGraph(k, voff, vls, q.src, q.dst, eoff, els, name=f"mlq{seed}")
