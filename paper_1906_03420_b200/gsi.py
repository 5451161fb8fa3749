"""Thin ctypes binding of libgsi_b200.so (include/gsi.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module converts numpy
arrays to pointers, fills the option structs and turns status codes into exceptions.  There
is no CPU fallback: if the shared library is missing the import fails loudly, and with no
CUDA device every compute call raises GsiError(GSI_ERR_CUDA).

The function names mirror the C ABI (gsi_build_graph, gsi_query, ...).  ``build``/``query``
are conveniences that take ``workloads.Graph``/``workloads.Query``-shaped objects.
"""
from __future__ import annotations

import ctypes
import os
import re
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GSI_LIB") or os.path.join(_PKG, "lib", "libgsi_b200.so")   # GSI_LIB: A/B builds
HEADER = os.path.join(os.path.dirname(_PKG), "include", "gsi.h")

GSI_MAX_K = 32
GSI_N_KCLASS = 8
KCLASS = ["filter", "compact", "probe", "join", "link", "other", "r6", "r7"]
GSI_N_KVARIANT = 20
ABL_ENGINE, ABL_CR, ABL_TWO_STEP, ABL_NO_WCACHE, ABL_NAIVE_SO, ABL_NO_LB, ABL_NO_DR = 1, 2, 4, 8, 16, 32, 64
KVARIANT = ["join_next", "join_count", "join_table", "join_cahead", "count_fast", "next_lean", "cahead_warp",
            "cahead_lean", "final_lean", "final_fp", "filter_partition", "refilter", "probe_ahead", "small",
            "two_step", "ablation", "final_table", "surv_scan", "fp_terms", "reserved19"]
STATUS = {0: "GSI_OK", -1: "GSI_ERR_INVALID_ARG", -2: "GSI_ERR_VERTEX_RANGE", -3: "GSI_ERR_LABEL_RANGE",
          -4: "GSI_ERR_SELF_LOOP", -5: "GSI_ERR_DUPLICATE_EDGE", -6: "GSI_ERR_QUERY_DISCONNECTED",
          -7: "GSI_ERR_QUERY_TOO_LARGE", -8: "GSI_ERR_OOM", -9: "GSI_ERR_TIMEOUT", -10: "GSI_ERR_CUDA",
          -11: "GSI_ERR_INTERNAL"}

P = ctypes.c_void_p
I32, I64, U32, U64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64


class gsi_build_opts(ctypes.Structure):
    _fields_ = [("gpn", I32), ("device", I32), ("stream", P)]


class gsi_query_opts(ctypes.Structure):
    _fields_ = [("want_table", I32), ("homomorphism", I32), ("filter_mode", I32), ("e0_mode", I32),
                ("force_order", P), ("force_first_edge", P), ("roots", P), ("n_roots", I64),
                ("shard_rank", I32), ("shard_count", I32), ("shard_min_rows", U64),
                ("mem_budget_bytes", U64), ("timeout_s", ctypes.c_double), ("profile", I32), ("stream", P),
                ("chunk_slots", U64), ("partial_on_timeout", I32), ("fingerprint", I32), ("no_shared_lists", I32),
                ("no_count_ahead", I32), ("shard_pieces", I32), ("force_paths", I32),
                ("small_mode", I32), ("ablation", I32)]


class gsi_graph_info(ctypes.Structure):
    _fields_ = [("n", I64), ("m", I64), ("n_elabels", I32), ("gpn", I32), ("n_groups", I64),
                ("max_chain", I32), ("overflow_groups", I64), ("bytes_groups", U64), ("bytes_ci", U64),
                ("bytes_sig", U64), ("bytes_total", U64), ("device", I32), ("ms_build", ctypes.c_float)]


class gsi_buffer_desc(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("dev_ptr", P), ("bytes", U64)]


class gsi_stats(ctypes.Structure):
    _fields_ = [("k", I32), ("levels", I32), ("order", I32 * GSI_MAX_K), ("cand", I64 * GSI_MAX_K),
                ("rows", U64 * GSI_MAX_K), ("gba", U64 * GSI_MAX_K), ("list_elems", U64 * GSI_MAX_K),
                ("n_edges", I32 * GSI_MAX_K), ("first_edge", I32 * GSI_MAX_K), ("count", U64),
                ("shard_level", I32), ("shard_row_begin", U64), ("shard_row_end", U64),
                ("ms_total", ctypes.c_float), ("ms_filter", ctypes.c_float), ("ms_plan", ctypes.c_float),
                ("ms_join", ctypes.c_float), ("ms_kernel", ctypes.c_float * GSI_N_KCLASS),
                ("launches", U32 * GSI_N_KCLASS), ("alg_bytes", ctypes.c_double * GSI_N_KCLASS),
                ("total_launches", U32), ("n_chunks", U32), ("capped", I32), ("h2d_bytes", U64),
                ("d2h_bytes", U64), ("n_shared_lists", U32), ("ms_host_alloc", ctypes.c_float),
                ("ms_host_sync", ctypes.c_float), ("count_ahead", I32), ("n_probe_ahead", U32),
                ("variant_launches", U32 * GSI_N_KVARIANT), ("ms_variant", ctypes.c_float * GSI_N_KVARIANT),
                ("alg_bytes_variant", ctypes.c_double * GSI_N_KVARIANT), ("small_aborted", I32),
                ("abl_layer_rows", U64 * 3), ("items_variant", U64 * GSI_N_KVARIANT)]


_SIGS = {
    "gsi_build_opts_default": (None, [P]),
    "gsi_query_opts_default": (None, [P]),
    "gsi_build_graph": (I32, [I64, P, I64, P, P, P, P, P]),
    "gsi_graph_info_get": (I32, [P, P]),
    "gsi_graph_buffers": (I32, [P, P, P, P, P]),
    "gsi_graph_alloc_like": (I32, [P, U64, P, P, P, P]),
    "gsi_graph_free": (None, [P]),
    "gsi_query": (I32, [P, I32, P, I32, P, P, P, P, P]),
    "gsi_query_prepare": (I32, [P, I32, P, I32, P, P, P, P]),
    "gsi_query_run": (I32, [P, P, P, P]),
    "gsi_prepared_free": (None, [P]),
    "gsi_result_count": (I32, [P, P]),
    "gsi_result_fingerprint": (I32, [P, P]),
    "gsi_trim_workspace": (None, [I32]),
    "gsi_query_run_batch": (I32, [P, I32, P, P, I32, P]),
    "gsi_result_table": (I32, [P, P, P]),
    "gsi_result_copy_table": (I32, [P, P, U64]),
    "gsi_result_stats": (I32, [P, P]),
    "gsi_result_free": (None, [P]),
    "gsi_debug_lookup": (I32, [P, I64, P, P, P, P, P, I64]),
    "gsi_debug_signatures": (I32, [P, P]),
    "gsi_debug_filter": (I32, [P, I32, P, I32, P, P, P, I32, P, P]),
    "gsi_debug_query_signatures": (I32, [I32, P, I32, P, P, P, I32, P]),
    "gsi_debug_hash": (U64, [I32, U64, U64]),
    "gsi_build_graph_ml": (I32, [I64, P, P, I64, P, P, P, P, P, P]),
    "gsi_build_line_graph": (I32, [I64, P, I64, P, P, P, P, P]),
    "gsi_query_prepare_ml": (I32, [P, I32, P, P, I32, P, P, P, P, P]),
    "gsi_query_prepare_line": (I32, [P, I32, P, I32, P, P, P, P]),
    "gsi_debug_filter_prepared": (I32, [P, I32, P, P]),
    "gsi_last_error": (ctypes.c_char_p, []),
    "gsi_version": (ctypes.c_char_p, []),
    "gsi_device_count": (I32, []),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def header_symbols() -> List[str]:
    """Every function the C header declares."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gsi_[a-z_0-9]+)\s*\(", txt)))


class GsiError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = (lib.gsi_last_error() or b"").decode()
        super().__init__(f"{where}: {STATUS.get(code, code)} ({msg})")
        self.code = code
        self.status = STATUS.get(code, str(code))


def _check(code: int, where: str):
    if code != 0:
        raise GsiError(code, where)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(P)


# ---------------------------------------------------------------------------- graph --
class GraphHandle:
    def __init__(self, h: int, keep=()):
        self.h = h
        self._keep = keep

    def __del__(self):
        h = getattr(self, "h", None)
        if h and lib is not None:
            lib.gsi_graph_free(h)
            self.h = None

    def info(self) -> Dict:
        return gsi_graph_info_get(self)


def gsi_build_graph(n: int, vlabels, src, dst, elabels, gpn: int = 16, device: int = -1, stream=None) -> GraphHandle:
    vl, s, d, e = _i32(vlabels), _i32(src), _i32(dst), _i32(elabels)
    if not (len(s) == len(d) == len(e)):
        raise ValueError("src/dst/elabels length mismatch")
    o = gsi_build_opts()
    lib.gsi_build_opts_default(ctypes.byref(o))
    o.gpn, o.device, o.stream = gpn, device, stream
    out = P()
    _check(lib.gsi_build_graph(n, _ptr(vl), len(s), _ptr(s), _ptr(d), _ptr(e), ctypes.byref(o), ctypes.byref(out)),
           "gsi_build_graph")
    return GraphHandle(out.value)


def _opts_build(gpn, device, stream):
    o = gsi_build_opts()
    lib.gsi_build_opts_default(ctypes.byref(o))
    o.gpn, o.device, o.stream = gpn, device, stream
    return o


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def gsi_build_graph_ml(n: int, vls_off, vls, src, dst, els_off, els, gpn: int = 16, device: int = -1,
                       stream=None) -> GraphHandle:
    """Multi-label graph (vertex and edge label SETS as offsets + labels), NEXT-4."""
    vo, vl, s, d, eo, el = _i64(vls_off), _i32(vls), _i32(src), _i32(dst), _i64(els_off), _i32(els)
    if len(vo) != n + 1 or len(eo) != len(s) + 1 or len(s) != len(d):
        raise ValueError("label-set offsets / edge arrays have inconsistent lengths")
    o = _opts_build(gpn, device, stream)
    out = P()
    _check(lib.gsi_build_graph_ml(n, _ptr(vo), _ptr(vl), len(s), _ptr(s), _ptr(d), _ptr(eo), _ptr(el),
                                  ctypes.byref(o), ctypes.byref(out)), "gsi_build_graph_ml")
    return GraphHandle(out.value)


def gsi_build_line_graph(n: int, vlabels, src, dst, elabels, gpn: int = 16, device: int = -1,
                         stream=None) -> GraphHandle:
    """Line graph for edge isomorphism (NEXT-4): vertex i = input edge i."""
    vl, s, d, e = _i32(vlabels), _i32(src), _i32(dst), _i32(elabels)
    if not (len(s) == len(d) == len(e)):
        raise ValueError("src/dst/elabels length mismatch")
    o = _opts_build(gpn, device, stream)
    out = P()
    _check(lib.gsi_build_line_graph(n, _ptr(vl), len(s), _ptr(s), _ptr(d), _ptr(e), ctypes.byref(o),
                                    ctypes.byref(out)), "gsi_build_line_graph")
    return GraphHandle(out.value)


def gsi_graph_info_get(g: GraphHandle) -> Dict:
    info = gsi_graph_info()
    _check(lib.gsi_graph_info_get(g.h, ctypes.byref(info)), "gsi_graph_info_get")
    return {f: getattr(info, f) for f, _ in gsi_graph_info._fields_}


def gsi_graph_buffers(g: GraphHandle) -> Tuple[List[Tuple[str, int, int]], bytes]:
    descs = (gsi_buffer_desc * 8)()
    nd = I32(0)
    mb = U64(0)
    _check(lib.gsi_graph_buffers(g.h, descs, ctypes.byref(nd), None, ctypes.byref(mb)), "gsi_graph_buffers")
    meta = ctypes.create_string_buffer(mb.value)
    _check(lib.gsi_graph_buffers(g.h, descs, ctypes.byref(nd), meta, ctypes.byref(mb)), "gsi_graph_buffers")
    return [(descs[i].name.decode(), descs[i].dev_ptr or 0, descs[i].bytes) for i in range(nd.value)], meta.raw


def gsi_graph_alloc_like(meta: bytes, device: int = -1) -> Tuple[GraphHandle, List[Tuple[str, int, int]]]:
    o = gsi_build_opts()
    lib.gsi_build_opts_default(ctypes.byref(o))
    o.device = device
    out = P()
    descs = (gsi_buffer_desc * 8)()
    nd = I32(0)
    buf = ctypes.create_string_buffer(meta, len(meta))
    _check(lib.gsi_graph_alloc_like(buf, len(meta), ctypes.byref(o), ctypes.byref(out), descs, ctypes.byref(nd)),
           "gsi_graph_alloc_like")
    return GraphHandle(out.value), [(descs[i].name.decode(), descs[i].dev_ptr or 0, descs[i].bytes)
                                    for i in range(nd.value)]


# ---------------------------------------------------------------------------- query --
class Result:
    def __init__(self, h: int, k: int):
        self.h = h
        self.k = k

    def __del__(self):
        h = getattr(self, "h", None)
        if h and lib is not None:
            lib.gsi_result_free(h)
            self.h = None

    @property
    def count(self) -> int:
        c = U64(0)
        _check(lib.gsi_result_count(self.h, ctypes.byref(c)), "gsi_result_count")
        return int(c.value)

    def fingerprint(self) -> Tuple[int, int, int]:
        fp = (U64 * 3)()
        _check(lib.gsi_result_fingerprint(self.h, fp), "gsi_result_fingerprint")
        return int(fp[0]), int(fp[1]), int(fp[2])

    def table_device(self) -> Tuple[int, int]:
        ptr, n = P(), U64(0)
        _check(lib.gsi_result_table(self.h, ctypes.byref(ptr), ctypes.byref(n)), "gsi_result_table")
        return ptr.value or 0, int(n.value)

    def table(self) -> np.ndarray:
        _, n = self.table_device()
        out = np.empty((max(n, 1), self.k), np.int32)
        _check(lib.gsi_result_copy_table(self.h, _ptr(out), n), "gsi_result_copy_table")
        return out[:n]

    def stats(self) -> Dict:
        s = gsi_stats()
        _check(lib.gsi_result_stats(self.h, ctypes.byref(s)), "gsi_result_stats")
        d = {}
        for f, _ in gsi_stats._fields_:
            v = getattr(s, f)
            d[f] = list(v) if hasattr(v, "__len__") else v
        d["variants"] = {KVARIANT[i]: d["variant_launches"][i] for i in range(GSI_N_KVARIANT)
                         if d["variant_launches"][i]}
        return d


class Prepared:
    def __init__(self, h: int, k: int, graph: "GraphHandle" = None):
        self.h = h
        self.k = k
        self.graph = graph   # the C handle points at its graph: keep the graph alive

    def __del__(self):
        h = getattr(self, "h", None)
        if h and lib is not None:
            lib.gsi_prepared_free(h)
            self.h = None


def _opts(want_table=False, homomorphism=False, filter_mode=0, e0_mode=0, force_order=None,
          force_first_edge=None, roots=None, shard_rank=0, shard_count=1, shard_min_rows=0,
          mem_budget_bytes=0, timeout_s=0.0, profile=False, stream=None, chunk_slots=0,
          partial_on_timeout=False, fingerprint=True, shared_lists=True, count_ahead=True, shard_pieces=1,
          force_paths=0, small=True, ablation=0):
    o = gsi_query_opts()
    lib.gsi_query_opts_default(ctypes.byref(o))
    keep = []
    o.want_table, o.homomorphism, o.filter_mode, o.e0_mode = int(want_table), int(homomorphism), filter_mode, e0_mode
    if force_order is not None:
        a = _i32(force_order); keep.append(a); o.force_order = _ptr(a)
    if force_first_edge is not None:
        a = _i32(force_first_edge); keep.append(a); o.force_first_edge = _ptr(a)
    if roots is not None:
        a = _i32(roots); keep.append(a); o.roots = _ptr(a); o.n_roots = len(a)
    o.shard_rank, o.shard_count, o.shard_min_rows = shard_rank, shard_count, shard_min_rows
    o.mem_budget_bytes, o.timeout_s, o.profile = mem_budget_bytes, timeout_s, int(profile)
    o.stream = stream
    o.chunk_slots, o.partial_on_timeout = chunk_slots, int(partial_on_timeout)
    o.fingerprint = int(fingerprint)   # binding default: on (the C default is off)
    o.no_shared_lists = 0 if shared_lists else 1
    o.no_count_ahead = 0 if count_ahead else 1
    o.shard_pieces = shard_pieces
    o.force_paths = force_paths
    o.small_mode = 0 if small else 1
    o.ablation = ablation
    return o, keep


def gsi_query(g: GraphHandle, q_vlabels, q_src, q_dst, q_elabels, **opts) -> Result:
    qv, qs, qd, qe = _i32(q_vlabels), _i32(q_src), _i32(q_dst), _i32(q_elabels)
    o, keep = _opts(**opts)
    out = P()
    _check(lib.gsi_query(g.h, len(qv), _ptr(qv), len(qs), _ptr(qs), _ptr(qd), _ptr(qe), ctypes.byref(o),
                         ctypes.byref(out)), "gsi_query")
    return Result(out.value, len(qv))


def gsi_query_prepare(g: GraphHandle, q_vlabels, q_src, q_dst, q_elabels) -> Prepared:
    qv, qs, qd, qe = _i32(q_vlabels), _i32(q_src), _i32(q_dst), _i32(q_elabels)
    out = P()
    _check(lib.gsi_query_prepare(g.h, len(qv), _ptr(qv), len(qs), _ptr(qs), _ptr(qd), _ptr(qe), ctypes.byref(out)),
           "gsi_query_prepare")
    return Prepared(out.value, len(qv), g)


def gsi_query_prepare_ml(g: GraphHandle, q_vls_off, q_vls, q_src, q_dst, q_els_off, q_els) -> Prepared:
    vo, vl, qs, qd, eo, el = _i32(q_vls_off), _i32(q_vls), _i32(q_src), _i32(q_dst), _i32(q_els_off), _i32(q_els)
    k = len(vo) - 1
    out = P()
    _check(lib.gsi_query_prepare_ml(g.h, k, _ptr(vo), _ptr(vl), len(qs), _ptr(qs), _ptr(qd), _ptr(eo), _ptr(el),
                                    ctypes.byref(out)), "gsi_query_prepare_ml")
    return Prepared(out.value, k, g)


def gsi_query_prepare_line(g: GraphHandle, q_vlabels, q_src, q_dst, q_elabels) -> Prepared:
    """Edge-isomorphism query: result rows hold one data edge id per query edge."""
    qv, qs, qd, qe = _i32(q_vlabels), _i32(q_src), _i32(q_dst), _i32(q_elabels)
    out = P()
    _check(lib.gsi_query_prepare_line(g.h, len(qv), _ptr(qv), len(qs), _ptr(qs), _ptr(qd), _ptr(qe),
                                      ctypes.byref(out)), "gsi_query_prepare_line")
    return Prepared(out.value, len(qs), g)


def gsi_query_run(g: GraphHandle, p: Prepared, **opts) -> Result:
    o, keep = _opts(**opts)
    out = P()
    _check(lib.gsi_query_run(g.h, p.h, ctypes.byref(o), ctypes.byref(out)), "gsi_query_run")
    return Result(out.value, p.k)


def gsi_query_run_batch(g: GraphHandle, prepared: Sequence["Prepared"], concurrency: int = 4, **opts) -> List[Result]:
    """Run prepared queries concurrently (`concurrency` host workers / streams)."""
    n = len(prepared)
    o, keep = _opts(**opts)
    arr = (P * max(n, 1))(*[p.h for p in prepared])
    outs = (P * max(n, 1))()
    _check(lib.gsi_query_run_batch(g.h, n, arr, ctypes.byref(o), int(concurrency), outs), "gsi_query_run_batch")
    return [Result(outs[i], prepared[i].k) for i in range(n)]


# ---------------------------------------------------------------------------- debug --
def gsi_debug_lookup(g: GraphHandle, v: Sequence[int], l: Sequence[int]):
    va, la = _i32(v), _i32(l)
    nq = len(va)
    lens = np.zeros(max(nq, 1), np.int64)
    reads = np.zeros(max(nq, 1), np.int32)
    _check(lib.gsi_debug_lookup(g.h, nq, _ptr(va), _ptr(la), _ptr(lens), _ptr(reads), None, 0), "gsi_debug_lookup")
    total = int(lens[:nq].sum())
    nb = np.zeros(max(total, 1), np.int32)
    _check(lib.gsi_debug_lookup(g.h, nq, _ptr(va), _ptr(la), _ptr(lens), _ptr(reads), _ptr(nb), total),
           "gsi_debug_lookup")
    return lens[:nq], reads[:nq], nb[:total]


def gsi_debug_signatures(g: GraphHandle) -> np.ndarray:
    n = gsi_graph_info_get(g)["n"]
    out = np.zeros((16, max(n, 1)), np.uint32)
    _check(lib.gsi_debug_signatures(g.h, _ptr(out)), "gsi_debug_signatures")
    return out[:, :n]


def gsi_debug_filter(g: GraphHandle, q_vlabels, q_src, q_dst, q_elabels, filter_mode: int = 0):
    qv, qs, qd, qe = _i32(q_vlabels), _i32(q_src), _i32(q_dst), _i32(q_elabels)
    n = gsi_graph_info_get(g)["n"]
    words = (n + 31) // 32
    bm = np.zeros((len(qv), max(words, 1)), np.uint32)
    cnt = np.zeros(len(qv), np.int64)
    _check(lib.gsi_debug_filter(g.h, len(qv), _ptr(qv), len(qs), _ptr(qs), _ptr(qd), _ptr(qe), filter_mode,
                                _ptr(bm), _ptr(cnt)), "gsi_debug_filter")
    return bm[:, :words], cnt


def gsi_debug_filter_prepared(p: Prepared, n: int, mode: int = 0):
    words = (n + 31) // 32
    bm = np.zeros((p.k, max(words, 1)), np.uint32)
    cnt = np.zeros(p.k, np.int64)
    _check(lib.gsi_debug_filter_prepared(p.h, mode, _ptr(bm), _ptr(cnt)), "gsi_debug_filter_prepared")
    return bm[:, :words], cnt


def gsi_debug_query_signatures(q_vlabels, q_src, q_dst, q_elabels, distinct: bool = False) -> np.ndarray:
    qv, qs, qd, qe = _i32(q_vlabels), _i32(q_src), _i32(q_dst), _i32(q_elabels)
    out = np.zeros((len(qv), 16), np.uint32)
    _check(lib.gsi_debug_query_signatures(len(qv), _ptr(qv), len(qs), _ptr(qs), _ptr(qd), _ptr(qe), int(distinct),
                                          _ptr(out)),
           "gsi_debug_query_signatures")
    return out


def gsi_debug_hash(kind: int, key: int, seed: int = 0) -> int:
    return int(lib.gsi_debug_hash(kind, key & 0xFFFFFFFFFFFFFFFF, seed & 0xFFFFFFFFFFFFFFFF))


def gsi_trim_workspace(device: int = -1) -> None:
    lib.gsi_trim_workspace(device)


def gsi_last_error() -> str:
    return (lib.gsi_last_error() or b"").decode()


def gsi_version() -> str:
    return lib.gsi_version().decode()


def gsi_device_count() -> int:
    return int(lib.gsi_device_count())


class _CudaArray:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def torch_view(ptr: int, nbytes: int, device=None):
    """Zero-copy torch.uint8 view of a library-owned device buffer (for NCCL broadcast of the
    graph arrays; torch is only plumbing here)."""
    import torch
    return torch.as_tensor(_CudaArray(ptr, nbytes), device=device if device is not None else "cuda")


# ------------------------------------------------------------------ conveniences ----
def build(g, gpn: int = 16, device: int = -1, stream=None) -> GraphHandle:
    return gsi_build_graph(g.n, g.vlabels, g.src, g.dst, g.elabels, gpn=gpn, device=device, stream=stream)


def query(graph: GraphHandle, q, **opts) -> Result:
    return gsi_query(graph, q.vlabels, q.src, q.dst, q.elabels, **opts)


def prepare(graph: GraphHandle, q) -> Prepared:
    return gsi_query_prepare(graph, q.vlabels, q.src, q.dst, q.elabels)


def build_ml(g, gpn: int = 16, device: int = -1, stream=None) -> GraphHandle:
    return gsi_build_graph_ml(g.n, g.vls_off, g.vls, g.src, g.dst, g.els_off, g.els, gpn=gpn, device=device,
                              stream=stream)


def prepare_ml(graph: GraphHandle, q) -> Prepared:
    return gsi_query_prepare_ml(graph, q.vls_off, q.vls, q.src, q.dst, q.els_off, q.els)


def query_ml(graph: GraphHandle, q, **opts) -> Result:
    return gsi_query_run(graph, prepare_ml(graph, q), **opts)


def build_line(g, gpn: int = 16, device: int = -1, stream=None) -> GraphHandle:
    return gsi_build_line_graph(g.n, g.vlabels, g.src, g.dst, g.elabels, gpn=gpn, device=device, stream=stream)


def prepare_line(graph: GraphHandle, q) -> Prepared:
    return gsi_query_prepare_line(graph, q.vlabels, q.src, q.dst, q.elabels)


def query_line(graph: GraphHandle, q, **opts) -> Result:
    return gsi_query_run(graph, prepare_line(graph, q), **opts)
