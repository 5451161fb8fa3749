"""CPU oracle for the GSI hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1906_03420_b200``) never imports it and shares no code with it.

Two independent matchers, each citing the definition it follows:

* ``match``        — the C backtracker in ``oracle.c`` (Fig. 2; Def. 2-3).
* ``brute_force``  — enumerate every injective map V(Q) -> V(G) for tiny inputs and keep
                     those that satisfy Def. 2's first two bullets;
                     it pins the backtracker.

plus the signature-filter specification (§III-A) in
``signatures`` / ``query_signatures`` / ``filter`` and the set fingerprint of SURVEY.md §8(c).
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ERRORS = {-1: "invalid argument", -2: "vertex out of range", -3: "label out of range",
          -4: "self loop", -5: "duplicate edge", -6: "query disconnected", -7: "query too large",
          -9: "timeout"}


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, OpenMP) into liboracle.so next to it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.og_build.restype = P
        L.og_build.argtypes = [I64, P, I64, P, P, P, P]
        L.og_free.argtypes = [P]
        L.og_match.restype = I64
        L.og_match.argtypes = [P, I32, P, I32, P, P, P, I32, P, I64, I32, I32, P, I64, P, ctypes.c_double]
        L.og_neighbors.restype = I64
        L.og_neighbors.argtypes = [P, I32, I32, P, I64]
        L.og_degree.restype = I64
        L.og_degree.argtypes = [P, I32]
        L.og_signatures.argtypes = [P, P]
        L.og_query_signatures.argtypes = [I32, P, I32, P, P, P, I32, P]
        L.og_filter.argtypes = [P, P, I32, P, P, P]
        L.og_fingerprint_rows.argtypes = [P, I64, I32, P]
        L.og_sig_group_of.restype = I32
        L.og_sig_group_of.argtypes = [I32, I32]
        L.og_max_threads.restype = I32
        L.og_murmur2_bytes.restype = ctypes.c_uint32
        L.og_murmur2_bytes.argtypes = [P, I64, ctypes.c_uint32]
        L.og_murmur64a_bytes.restype = ctypes.c_uint64
        L.og_murmur64a_bytes.argtypes = [P, I64, ctypes.c_uint64]
        L.og_smhasher_verify.restype = ctypes.c_uint32
        L.og_smhasher_verify.argtypes = [I32]
        L.og_set_label_sets.restype = I32
        L.og_set_label_sets.argtypes = [P, P, P]
        L.og_match_ml.restype = I64
        L.og_match_ml.argtypes = [P, I32, P, P, I32, P, P, P, I32, P, I64, I32, I32, P, I64, P, ctypes.c_double]
        L.og_match_edges.restype = I64
        L.og_match_edges.argtypes = [P, P, P, P, I32, P, I32, P, P, P, P, I64, P, ctypes.c_double]
        L.og_signatures_ml.argtypes = [P, P]
        L.og_query_signatures_ml.argtypes = [I32, P, P, I32, P, P, P, I32, P]
        L.og_filter_ml.argtypes = [P, P, I32, P, P, P, P, P]
        L.og_murmur64a_key.restype = ctypes.c_uint64
        L.og_murmur64a_key.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle error {code}: {ERRORS.get(code, '?')}")
        self.code = code


class OracleGraph:
    """The oracle's own index of G: per-vertex adjacency sorted by (edge label, neighbour)."""

    def __init__(self, g):
        self.n = int(g.n)
        self._vl, self._s, self._d, self._e = _i32(g.vlabels), _i32(g.src), _i32(g.dst), _i32(g.elabels)
        err = ctypes.c_int32(0)
        self._h = lib().og_build(self.n, _p(self._vl), len(self._s), _p(self._s), _p(self._d), _p(self._e),
                                 ctypes.byref(err))
        if not self._h:
            raise OracleError(err.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            try:
                _lib.og_free(h)
            except Exception:
                pass
            self._h = None

    def neighbors(self, v: int, l: int) -> np.ndarray:
        """N(v,l) ascending."""
        cnt = lib().og_neighbors(self._h, v, l, None, 0)
        out = np.empty(max(cnt, 1), np.int32)
        lib().og_neighbors(self._h, v, l, _p(out), cnt)
        return out[:cnt]

    def degree(self, v: int) -> int:
        return int(lib().og_degree(self._h, v))


def match(og: OracleGraph, q, root: int = 0, roots: Optional[Sequence[int]] = None, threads: int = 0,
          hom: bool = False, table: bool = True, cap: Optional[int] = None,
          timeout: float = 0.0, partial: bool = False) -> Tuple[int, Tuple[int, int, int], Optional[np.ndarray]]:
    """Enumerate R(Q,G).  Returns (count, fingerprint (count, sum, xor), table or None);
    the table is k int32 per row in query-id order, sorted lexicographically.
    partial=True (count-only): on timeout return the matches found so far instead of raising."""
    qv, qs, qd, qe = _i32(q.vlabels), _i32(q.src), _i32(q.dst), _i32(q.elabels)
    r = None if roots is None else _i32(roots)
    fp = np.zeros(3, np.uint64)
    k = int(q.n)
    if table:
        if cap is None:
            cnt = lib().og_match(og._h, k, _p(qv), len(qs), _p(qs), _p(qd), _p(qe), root,
                                 None if r is None else _p(r), 0 if r is None else len(r), threads,
                                 int(hom), None, 0, _p(fp), timeout)
            if cnt < 0:
                raise OracleError(int(cnt))
            cap = cnt
        out = np.empty((max(cap, 1), k), np.int32)
    else:
        out = None
    cnt = lib().og_match(og._h, k, _p(qv), len(qs), _p(qs), _p(qd), _p(qe), root,
                         None if r is None else _p(r), 0 if r is None else len(r), threads, int(hom),
                         None if out is None else _p(out), 0 if out is None else cap, _p(fp), timeout)
    if cnt == -9 and partial and out is None:
        cnt = int(fp[0])
    elif cnt < 0:
        raise OracleError(int(cnt))
    fpt = (int(fp[0]), int(fp[1]), int(fp[2]))
    return int(cnt), fpt, (None if out is None else out[: min(cnt, cap)])


def fingerprint_rows(rows: np.ndarray, k: int) -> Tuple[int, int, int]:
    rows = _i32(rows).reshape(-1, k)
    fp = np.zeros(3, np.uint64)
    lib().og_fingerprint_rows(_p(rows), rows.shape[0], k, _p(fp))
    return int(fp[0]), int(fp[1]), int(fp[2])


# ------------------------------------------------------------------ signatures ----
def signatures(og: OracleGraph) -> np.ndarray:
    """Column-first data signature table, shape (16, n) uint32."""
    planes = np.zeros((16, og.n), np.uint32)
    lib().og_signatures(og._h, _p(planes))
    return planes


def query_signatures(q, distinct: bool = False) -> np.ndarray:
    """Query signatures, shape (k, 16) uint32 (PAPER.md L545 'same encoding strategy');
    distinct=True is the homomorphism encoding (each pair counted once)."""
    out = np.zeros((q.n, 16), np.uint32)
    lib().og_query_signatures(q.n, _p(_i32(q.vlabels)), len(q.src), _p(_i32(q.src)), _p(_i32(q.dst)),
                              _p(_i32(q.elabels)), int(distinct), _p(out))
    return out


def filter(og: OracleGraph, planes: np.ndarray, qsig: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """C(u) bitmaps (k, ceil(n/32)) uint32 and |C(u)| (k,) int64 (reading A4)."""
    k = qsig.shape[0]
    words = (og.n + 31) // 32
    bm = np.zeros((k, max(words, 1)), np.uint32)
    cnt = np.zeros(k, np.int64)
    lib().og_filter(og._h, _p(np.ascontiguousarray(planes)), k, _p(np.ascontiguousarray(qsig)), _p(bm), _p(cnt))
    return bm[:, :words], cnt


def sig_group(elabel: int, nlabel: int) -> int:
    return int(lib().og_sig_group_of(elabel, nlabel))


def murmur2(data: bytes, seed: int) -> int:
    """MurmurHash2 (32-bit) of a byte string (the oracle's general restatement)."""
    b = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
    return int(lib().og_murmur2_bytes(_p(b), len(data), seed & 0xFFFFFFFF))


def murmur64a(data: bytes, seed: int) -> int:
    """MurmurHash64A of a byte string (the oracle's general restatement)."""
    b = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
    return int(lib().og_murmur64a_bytes(_p(b), len(data), seed & 0xFFFFFFFFFFFFFFFF))


def murmur64a_key(key: int, seed: int) -> int:
    """The oracle's signature hash (8-byte specialisation used by og_sig_group)."""
    return int(lib().og_murmur64a_key(key, seed))


def smhasher_verify(which: int) -> int:
    """SMHasher's verification value of the general hash: 0 = MurmurHash2, 1 = MurmurHash64A."""
    return int(lib().og_smhasher_verify(which))


def max_threads() -> int:
    return int(lib().og_max_threads())


# ------------------------------------------------------------------ brute force ----
def brute_force(g, q, hom: bool = False) -> List[Tuple[int, ...]]:
    """All maps f: V(Q)->V(G) (injective unless hom) with L_V(f(u)) = L_V(u) and every query
    edge (a,b,l) present as a data edge {f(a),f(b)} labelled l (Def. 2 bullets 1-2,
    L278-279; Def. 3).  Pure Python; tiny inputs only (n <= 9, k <= 5)."""
    n, k = int(g.n), int(q.n)
    edges = set()
    for s, d, l in zip(g.src.tolist(), g.dst.tolist(), g.elabels.tolist()):
        edges.add((s, d, l)); edges.add((d, s, l))
    qe = list(zip(q.src.tolist(), q.dst.tolist(), q.elabels.tolist()))
    gl, ql = g.vlabels.tolist(), q.vlabels.tolist()
    it = itertools.product(range(n), repeat=k) if hom else itertools.permutations(range(n), k)
    out = []
    for f in it:
        if any(gl[f[u]] != ql[u] for u in range(k)):
            continue
        if all((f[a], f[b], l) in edges for a, b, l in qe):
            out.append(tuple(f))
    out.sort()
    return out


# ------------------------------------------------------------ multi-label (§VII-B) ----
def _expand_edges(src, dst, off, labs):
    """L_E(e) ⊆ L_E(f(e)) is a conjunction over the labels of e: one single-label edge per
    label (Fig. 10)."""
    cnt = np.diff(off)
    return (np.repeat(_i32(src), cnt), np.repeat(_i32(dst), cnt), _i32(labs))


class OracleMLGraph(OracleGraph):
    """The oracle's index of a multi-label graph: parallel single-label edges plus the
    vertex label SETS (og_set_label_sets)."""

    def __init__(self, g):
        self.n = int(g.n)
        s_, d_, e_ = _expand_edges(g.src, g.dst, g.els_off, g.els)
        self._vl, self._s, self._d, self._e = np.zeros(self.n, np.int32), s_, d_, e_
        err = ctypes.c_int32(0)
        self._h = lib().og_build(self.n, _p(self._vl), len(s_), _p(s_), _p(d_), _p(e_), ctypes.byref(err))
        if not self._h:
            raise OracleError(err.value)
        self._lo, self._ls = np.ascontiguousarray(g.vls_off, np.int64), _i32(g.vls)
        rc = lib().og_set_label_sets(self._h, _p(self._lo), _p(self._ls))
        if rc:
            raise OracleError(int(rc))


def match_ml(og: OracleMLGraph, q, hom: bool = False, table: bool = True, threads: int = 0,
             timeout: float = 0.0) -> Tuple[int, Tuple[int, int, int], Optional[np.ndarray]]:
    """R(Q,G) under the multi-label definition: f injective (unless hom),
    L_V(u) ⊆ L_V(f(u)), L_E(uv) ⊆ L_E(f(u)f(v)).  Same return shape as match()."""
    qs, qd, qe = _expand_edges(q.src, q.dst, q.els_off, q.els)
    qo = _i32(q.vls_off)
    ql = _i32(q.vls)
    fp = np.zeros(3, np.uint64)
    k = int(q.n)
    args = (og._h, k, _p(qo), _p(ql), len(qs), _p(qs), _p(qd), _p(qe), 0, None, 0, threads, int(hom))
    cnt = lib().og_match_ml(*args, None, 0, _p(fp), timeout)
    if cnt < 0:
        raise OracleError(int(cnt))
    out = None
    if table:
        out = np.empty((max(cnt, 1), k), np.int32)
        cnt = lib().og_match_ml(*args, _p(out), cnt, _p(fp), timeout)
        out = out[:cnt]
    return int(cnt), (int(fp[0]), int(fp[1]), int(fp[2])), out


def brute_force_ml(g, q, hom: bool = False) -> List[Tuple[int, ...]]:
    """Every map f with L_V(u) ⊆ L_V(f(u)) and L_E(ab) ⊆ L_E(f(a)f(b)) for every query edge
    (PAPER.md L1273-1275), injective unless hom.  Pure Python, tiny inputs."""
    n, k = int(g.n), int(q.n)
    eset = {}
    for i, (a, b) in enumerate(zip(g.src.tolist(), g.dst.tolist())):
        st = set(g.els[g.els_off[i]:g.els_off[i + 1]].tolist())
        eset.setdefault((a, b), set()).update(st)
        eset.setdefault((b, a), set()).update(st)
    vset = [set(g.vls[g.vls_off[v]:g.vls_off[v + 1]].tolist()) for v in range(n)]
    qv = [set(q.vls[q.vls_off[u]:q.vls_off[u + 1]].tolist()) for u in range(k)]
    qe = [(a, b, set(q.els[q.els_off[i]:q.els_off[i + 1]].tolist()))
          for i, (a, b) in enumerate(zip(q.src.tolist(), q.dst.tolist()))]
    it = itertools.product(range(n), repeat=k) if hom else itertools.permutations(range(n), k)
    out = []
    for f in it:
        if any(not qv[u] <= vset[f[u]] for u in range(k)):
            continue
        if all(ls <= eset.get((f[a], f[b]), set()) for a, b, ls in qe):
            out.append(tuple(f))
    out.sort()
    return out


def signatures_ml(og: OracleMLGraph) -> np.ndarray:
    """Multi-label data signatures (16, n) (reading A19: hashed label bits in plane 0)."""
    planes = np.zeros((16, og.n), np.uint32)
    lib().og_signatures_ml(og._h, _p(planes))
    return planes


def query_signatures_ml(q, distinct: bool = False) -> np.ndarray:
    qs, qd, qe = _expand_edges(q.src, q.dst, q.els_off, q.els)
    out = np.zeros((q.n, 16), np.uint32)
    lib().og_query_signatures_ml(q.n, _p(_i32(q.vls_off)), _p(_i32(q.vls)), len(qs), _p(qs), _p(qd), _p(qe),
                                 int(distinct), _p(out))
    return out


def filter_ml(og: OracleMLGraph, planes: np.ndarray, qsig: np.ndarray, q) -> Tuple[np.ndarray, np.ndarray]:
    """Refined C(u) (signature containment on all 16 planes + exact L_V(u) ⊆ L_V(v))."""
    k = qsig.shape[0]
    words = (og.n + 31) // 32
    bm = np.zeros((k, max(words, 1)), np.uint32)
    cnt = np.zeros(k, np.int64)
    lib().og_filter_ml(og._h, _p(np.ascontiguousarray(planes)), k, _p(np.ascontiguousarray(qsig)),
                       _p(_i32(q.vls_off)), _p(_i32(q.vls)), _p(bm), _p(cnt))
    return bm[:, :words], cnt


# ------------------------------------------------------------ edge isomorphism ------
def match_edges(og: OracleGraph, g, q, table: bool = True,
                timeout: float = 0.0) -> Tuple[int, Tuple[int, int, int], Optional[np.ndarray]]:
    """R_E(Q,G) (§VII-A, reading A18): injective maps of query edges to
    data edges with equal edge labels such that any two query edges sharing a vertex w map to
    data edges sharing a vertex labelled L_V(w).  Rows: the data edge index (position in g's
    edge list) of query edges 0..|E(Q)|-1, sorted."""
    qv, qs, qd, qe = _i32(q.vlabels), _i32(q.src), _i32(q.dst), _i32(q.elabels)
    gs, gd, ge = _i32(g.src), _i32(g.dst), _i32(g.elabels)
    fp = np.zeros(3, np.uint64)
    k = len(qs)
    args = (og._h, _p(gs), _p(gd), _p(ge), int(q.n), _p(qv), k, _p(qs), _p(qd), _p(qe))
    cnt = lib().og_match_edges(*args, None, 0, _p(fp), timeout)
    if cnt < 0:
        raise OracleError(int(cnt))
    out = None
    if table:
        out = np.empty((max(cnt, 1), k), np.int32)
        cnt = lib().og_match_edges(*args, _p(out), cnt, _p(fp), timeout)
        out = out[:cnt]
    return int(cnt), (int(fp[0]), int(fp[1]), int(fp[2])), out


def brute_force_edges(g, q) -> List[Tuple[int, ...]]:
    """Every injective h: E(Q) -> E(G) with L_E(h(e)) = L_E(e) and, for query edges e1 != e2
    sharing a vertex w, h(e1) and h(e2) sharing a vertex labelled L_V(w).  Tiny inputs."""
    ge = list(zip(g.src.tolist(), g.dst.tolist(), g.elabels.tolist()))
    qe = list(zip(q.src.tolist(), q.dst.tolist(), q.elabels.tolist()))
    gl, ql = g.vlabels.tolist(), q.vlabels.tolist()
    shared = []   # (i, j, label of a shared query vertex)
    for i in range(len(qe)):
        for j in range(i + 1, len(qe)):
            for w in set(qe[i][:2]) & set(qe[j][:2]):
                shared.append((i, j, ql[w]))
    out = []
    for h in itertools.permutations(range(len(ge)), len(qe)):
        if any(ge[h[i]][2] != qe[i][2] for i in range(len(qe))):
            continue
        if all(any(gl[v] == lab for v in set(ge[h[i]][:2]) & set(ge[h[j]][:2])) for i, j, lab in shared):
            out.append(tuple(h))
    out.sort()
    return out
