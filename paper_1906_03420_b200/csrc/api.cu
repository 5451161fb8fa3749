// api.cu — extern "C" entry points of libgsi_b200 (declared in include/gsi.h).
// Argument checking, error strings and handle ownership live here; the device work is in
// graph.cu (PCSR + signature build) and query.cu (filter, planner, join).
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "common.cuh"

namespace gsi {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
std::string gsi_last_error_str() { return g_last_error; }

gsi_status cuda_fail(cudaError_t e, const char *what) {
    g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? GSI_ERR_OOM : GSI_ERR_CUDA;
}

gsi_status build_graph_impl(int64_t n, const int32_t *vl, int64_t m, const int32_t *src, const int32_t *dst,
                            const int32_t *el, const gsi_build_opts *opts, gsi_graph **out);
gsi_status debug_lookup_impl(const gsi_graph *g, int64_t nq, const int32_t *v, const int32_t *l, int64_t *len,
                             int32_t *groups_read, int32_t *nbrs, int64_t cap);
gsi_status prepare_impl(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                        const int32_t *qd, const int32_t *qe, gsi_prepared **out);
gsi_status run_impl(const gsi_graph *g, const gsi_prepared *q, const gsi_query_opts *opts, gsi_result **out);
gsi_status run_batch_impl(const gsi_graph *g, int32_t nq, const gsi_prepared *const *qs, const gsi_query_opts *opts,
                          int32_t conc, gsi_result **out);
gsi_status build_graph_ml_impl(int64_t n, const int64_t *vls_off, const int32_t *vls, int64_t m, const int32_t *src,
                               const int32_t *dst, const int64_t *els_off, const int32_t *els,
                               const gsi_build_opts *opts, gsi_graph **out);
gsi_status build_line_graph_impl(int64_t n, const int32_t *vl, int64_t m, const int32_t *src, const int32_t *dst,
                                 const int32_t *el, const gsi_build_opts *opts, gsi_graph **out);
gsi_status prepare_ml_impl(const gsi_graph *g, int32_t k, const int32_t *qvls_off, const int32_t *qvls, int32_t qm,
                           const int32_t *qs, const int32_t *qd, const int32_t *qels_off, const int32_t *qels,
                           gsi_prepared **out);
gsi_status prepare_line_impl(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                             const int32_t *qd, const int32_t *qe, gsi_prepared **out);
gsi_status debug_filter_prepared_impl(const gsi_prepared *q, int32_t mode, uint32_t *bitmaps, int64_t *counts);
gsi_status debug_filter_impl(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                             const int32_t *qd, const int32_t *qe, int32_t mode, uint32_t *bitmaps, int64_t *counts);

static gsi_status need_device() {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess || c == 0) {
        cudaGetLastError();
        g_last_error = "no CUDA device available (libgsi_b200 has no CPU path)";
        return GSI_ERR_CUDA;
    }
    return GSI_OK;
}

static void free_graph(gsi_graph *g) {
    if (!g) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(g->device);
    if (g->sig) cudaFree(g->sig);
    if (g->groups) cudaFree(g->groups);
    if (g->ci) cudaFree(g->ci);
    if (g->cr_key) cudaFree(g->cr_key);
    if (g->cr_loc) cudaFree(g->cr_loc);
    if (g->ml_off) cudaFree(g->ml_off);
    if (g->ml_labs) cudaFree(g->ml_labs);
    cudaSetDevice(cur);
    delete g;
}

struct MetaHeader {
    uint64_t magic;
    int64_t n, m, n_groups, overflow_groups;
    int32_t n_labels, gpn, max_chain, version;
    int64_t line_n;      // line graph (edge isomorphism): |V| of the original graph, else -1
};
static const uint64_t kMetaMagic = 0x475349423230304dull;   // "GSIB200M"

}  // namespace gsi

using namespace gsi;

extern "C" {

void gsi_build_opts_default(gsi_build_opts *o) {
    if (!o) return;
    o->gpn = 16;
    o->device = -1;
    o->stream = nullptr;
}

void gsi_trim_workspace(int32_t device) {
    int dev = device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    gsi::workspace_trim(dev);
}

void gsi_query_opts_default(gsi_query_opts *o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->shard_rank = 0;
    o->shard_count = 1;
}

gsi_status gsi_build_graph(int64_t n, const int32_t *vlabels, int64_t m, const int32_t *src, const int32_t *dst,
                           const int32_t *elabels, const gsi_build_opts *opts, gsi_graph **out) {
    if (!out) {
        set_error("out is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    GSI_TRY(need_device());
    gsi_build_opts o;
    gsi_build_opts_default(&o);
    if (opts) o = *opts;
    return build_graph_impl(n, vlabels, m, src, dst, elabels, &o, out);
}

gsi_status gsi_graph_info_get(const gsi_graph *g, gsi_graph_info *info) {
    if (!g || !info) {
        set_error("null argument");
        return GSI_ERR_INVALID_ARG;
    }
    std::memset(info, 0, sizeof(*info));
    info->n = g->n;
    info->m = g->m;
    info->n_elabels = g->n_labels;
    info->gpn = g->gpn;
    info->n_groups = g->n_groups;
    info->max_chain = g->max_chain;
    info->overflow_groups = g->overflow_groups;
    info->bytes_groups = (uint64_t)g->n_groups * g->gpn * 8;
    info->bytes_ci = (uint64_t)g->m * 8;
    info->bytes_sig = (uint64_t)g->n * kPlanes * 4;
    info->bytes_total = info->bytes_groups + info->bytes_ci + info->bytes_sig;
    info->device = g->device;
    info->ms_build = g->ms_build;
    return GSI_OK;
}

gsi_status gsi_graph_buffers(const gsi_graph *g, gsi_buffer_desc *descs, int32_t *ndesc, void *meta,
                             uint64_t *meta_bytes) {
    if (!g || !ndesc || !meta_bytes) {
        set_error("null argument");
        return GSI_ERR_INVALID_ARG;
    }
    if (g->ml) {
        set_error("replicating a multi-label graph is not supported (build it on every device)");
        return GSI_ERR_INVALID_ARG;
    }
    const int nl = g->n_labels;
    const uint64_t need = sizeof(MetaHeader) + (uint64_t)nl * (4 + 8 + 8 + 4) + 4ull * (nl + 1);
    if (descs) {
        descs[0] = {"sig", g->sig, (uint64_t)g->n * kPlanes * 4};
        descs[1] = {"groups", g->groups, (uint64_t)g->n_groups * g->gpn * 8};
        descs[2] = {"ci", g->ci, (uint64_t)g->m * 8};
    }
    *ndesc = 3;
    if (meta) {
        if (*meta_bytes < need) {
            set_error("meta buffer too small");
            return GSI_ERR_INVALID_ARG;
        }
        MetaHeader h{kMetaMagic, g->n, g->m, g->n_groups, g->overflow_groups, nl, g->gpn, g->max_chain, 3,
                     g->line ? g->line_n : -1};
        char *p = (char *)meta;
        std::memcpy(p, &h, sizeof(h));
        p += sizeof(h);
        std::memcpy(p, g->lab_raw.data(), 4ull * nl);
        p += 4ull * nl;
        std::memcpy(p, g->freq.data(), 8ull * nl);
        p += 8ull * nl;
        std::memcpy(p, g->gbase.data(), 8ull * nl);
        p += 8ull * nl;
        std::memcpy(p, g->ngroups.data(), 4ull * nl);
        p += 4ull * nl;
        std::memcpy(p, g->ci_lo.data(), 4ull * (nl + 1));
    }
    *meta_bytes = need;
    return GSI_OK;
}

gsi_status gsi_graph_alloc_like(const void *meta, uint64_t meta_bytes, const gsi_build_opts *opts, gsi_graph **out,
                                gsi_buffer_desc *descs, int32_t *ndesc) {
    if (!meta || !out || meta_bytes < sizeof(MetaHeader)) {
        set_error("invalid metadata");
        return GSI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    GSI_TRY(need_device());
    MetaHeader h;
    std::memcpy(&h, meta, sizeof(h));
    const int nl = h.n_labels;
    if (h.magic != kMetaMagic || h.version != 3 || meta_bytes < sizeof(MetaHeader) + (uint64_t)nl * 24 + 4ull * (nl + 1)) {
        set_error("metadata blob is not a gsi graph description");
        return GSI_ERR_INVALID_ARG;
    }
    if (opts && opts->device >= 0) GSI_CUDA(cudaSetDevice(opts->device));
    auto g = new gsi_graph();
    std::unique_ptr<gsi_graph, void (*)(gsi_graph *)> guard(g, free_graph);
    GSI_CUDA(cudaGetDevice(&g->device));
    g->n = h.n;
    g->m = h.m;
    g->n_groups = h.n_groups;
    g->overflow_groups = h.overflow_groups;
    g->n_labels = nl;
    g->gpn = h.gpn;
    g->max_chain = h.max_chain;
    g->line = h.line_n >= 0;
    g->line_n = g->line ? h.line_n : 0;
    const char *p = (const char *)meta + sizeof(h);
    g->lab_raw.resize(nl);
    g->freq.resize(nl);
    g->gbase.resize(nl);
    g->ngroups.resize(nl);
    std::memcpy(g->lab_raw.data(), p, 4ull * nl);
    p += 4ull * nl;
    std::memcpy(g->freq.data(), p, 8ull * nl);
    p += 8ull * nl;
    std::memcpy(g->gbase.data(), p, 8ull * nl);
    p += 8ull * nl;
    std::memcpy(g->ngroups.data(), p, 4ull * nl);
    p += 4ull * nl;
    g->ci_lo.resize(nl + 1);
    std::memcpy(g->ci_lo.data(), p, 4ull * (nl + 1));
    {
        int dev = 0;
        GSI_CUDA(cudaGetDevice(&dev));
        workspace_trim(dev);
    }
    GSI_CUDA(cudaMalloc(&g->sig, std::max<uint64_t>(16, (uint64_t)g->n * kPlanes * 4)));
    GSI_CUDA(cudaMalloc(&g->groups, std::max<uint64_t>(16, (uint64_t)g->n_groups * g->gpn * 8)));
    GSI_CUDA(cudaMalloc(&g->ci, std::max<uint64_t>(16, (uint64_t)g->m * 8)));
    if (descs) {
        descs[0] = {"sig", g->sig, (uint64_t)g->n * kPlanes * 4};
        descs[1] = {"groups", g->groups, (uint64_t)g->n_groups * g->gpn * 8};
        descs[2] = {"ci", g->ci, (uint64_t)g->m * 8};
    }
    if (ndesc) *ndesc = 3;
    *out = guard.release();
    return GSI_OK;
}

void gsi_graph_free(gsi_graph *g) { free_graph(g); }

gsi_status gsi_query_prepare(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                             const int32_t *qd, const int32_t *qe, gsi_prepared **out) {
    if (!out) {
        set_error("out is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    GSI_TRY(need_device());
    if (g && g->ml) {
        set_error("a multi-label graph takes gsi_query_prepare_ml");
        return GSI_ERR_INVALID_ARG;
    }
    return prepare_impl(g, k, qvl, qm, qs, qd, qe, out);
}

gsi_status gsi_query_prepare_ml(const gsi_graph *g, int32_t k, const int32_t *q_vls_off, const int32_t *q_vls,
                                int32_t qm, const int32_t *q_src, const int32_t *q_dst, const int32_t *q_els_off,
                                const int32_t *q_els, gsi_prepared **out) {
    if (!out) {
        set_error("out is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    GSI_TRY(need_device());
    return prepare_ml_impl(g, k, q_vls_off, q_vls, qm, q_src, q_dst, q_els_off, q_els, out);
}

gsi_status gsi_query_prepare_line(const gsi_graph *g, int32_t k, const int32_t *q_vlabels, int32_t qm,
                                  const int32_t *q_src, const int32_t *q_dst, const int32_t *q_elabels,
                                  gsi_prepared **out) {
    if (!out) {
        set_error("out is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    GSI_TRY(need_device());
    return prepare_line_impl(g, k, q_vlabels, qm, q_src, q_dst, q_elabels, out);
}

gsi_status gsi_build_graph_ml(int64_t n, const int64_t *vls_off, const int32_t *vls, int64_t m, const int32_t *src,
                              const int32_t *dst, const int64_t *els_off, const int32_t *els,
                              const gsi_build_opts *opts, gsi_graph **out) {
    if (!out) {
        set_error("out is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    GSI_TRY(need_device());
    return build_graph_ml_impl(n, vls_off, vls, m, src, dst, els_off, els, opts, out);
}

gsi_status gsi_build_line_graph(int64_t n, const int32_t *vlabels, int64_t m, const int32_t *src, const int32_t *dst,
                                const int32_t *elabels, const gsi_build_opts *opts, gsi_graph **out) {
    if (!out) {
        set_error("out is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    GSI_TRY(need_device());
    return build_line_graph_impl(n, vlabels, m, src, dst, elabels, opts, out);
}

gsi_status gsi_debug_filter_prepared(const gsi_prepared *q, int32_t mode, uint32_t *bitmaps, int64_t *counts) {
    GSI_TRY(need_device());
    if (!q) {
        set_error("q is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    return debug_filter_prepared_impl(q, mode, bitmaps, counts);
}

gsi_status gsi_query_run(const gsi_graph *g, const gsi_prepared *q, const gsi_query_opts *opts, gsi_result **out) {
    if (!out) {
        set_error("out is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    GSI_TRY(need_device());
    return run_impl(g, q, opts, out);
}

uint64_t gsi_debug_hash(int32_t kind, uint64_t key, uint64_t seed) {
    switch (kind) {
    case 0: return gsi::murmur2_u32((uint32_t)key, (uint32_t)seed);
    case 1: return gsi::murmur64a_u64(key, seed);
    case 2: return gsi::fp_mix(key);
    default: return 0;
    }
}

void gsi_prepared_free(gsi_prepared *q) {
    if (!q) return;
    cudaSetDevice(q->device);   // its device copy of the signatures lives on the graph's device
    delete q;
}

gsi_status gsi_query_run_batch(const gsi_graph *g, int32_t nq, const gsi_prepared *const *qs,
                               const gsi_query_opts *opts, int32_t concurrency, gsi_result **out) {
    if (nq > 0 && !out) {
        set_error("out is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    GSI_TRY(need_device());
    for (int i = 0; i < nq; i++)
        if (!qs || !qs[i] || qs[i]->g != g) {
            set_error("batch entry " + std::to_string(i) + " is not a query prepared for this graph");
            return GSI_ERR_INVALID_ARG;
        }
    return run_batch_impl(g, nq, qs, opts, concurrency, out);
}

gsi_status gsi_query(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                     const int32_t *qd, const int32_t *qe, const gsi_query_opts *opts, gsi_result **out) {
    if (!out) {
        set_error("out is NULL");
        return GSI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    GSI_TRY(need_device());
    gsi_prepared *p = nullptr;
    GSI_TRY(prepare_impl(g, k, qvl, qm, qs, qd, qe, &p));
    std::unique_ptr<gsi_prepared> guard(p);
    gsi_status rc = run_impl(g, p, opts, out);
    if (rc == GSI_OK) (*out)->stats.h2d_bytes += 4ull * p->qsig.size();   // encoded Q signatures (iso + hom)
    return rc;
}

gsi_status gsi_result_count(const gsi_result *r, uint64_t *count) {
    if (!r || !count) {
        set_error("null argument");
        return GSI_ERR_INVALID_ARG;
    }
    *count = r->count;
    return GSI_OK;
}

gsi_status gsi_result_fingerprint(const gsi_result *r, uint64_t fp[3]) {
    if (!r || !fp) {
        set_error("null argument");
        return GSI_ERR_INVALID_ARG;
    }
    fp[0] = r->fp[0];
    fp[1] = r->fp[1];
    fp[2] = r->fp[2];
    return GSI_OK;
}

gsi_status gsi_result_table(const gsi_result *r, const int32_t **dev_rows, uint64_t *nrows) {
    if (!r || !dev_rows || !nrows) {
        set_error("null argument");
        return GSI_ERR_INVALID_ARG;
    }
    if (!r->has_table) {
        set_error("query was run without want_table");
        return GSI_ERR_INVALID_ARG;
    }
    *dev_rows = r->table;
    *nrows = r->nrows;
    return GSI_OK;
}

gsi_status gsi_result_copy_table(const gsi_result *r, int32_t *host_rows, uint64_t cap) {
    if (!r || (!host_rows && cap)) {
        set_error("null argument");
        return GSI_ERR_INVALID_ARG;
    }
    if (!r->has_table) {
        set_error("query was run without want_table");
        return GSI_ERR_INVALID_ARG;
    }
    uint64_t rows = std::min<uint64_t>(cap, r->nrows);
    if (rows && r->table) {
        GSI_CUDA(cudaSetDevice(r->device));
        GSI_CUDA(cudaMemcpy(host_rows, r->table, 4ull * rows * r->k, cudaMemcpyDeviceToHost));
    }
    return GSI_OK;
}

gsi_status gsi_result_stats(const gsi_result *r, gsi_stats *s) {
    if (!r || !s) {
        set_error("null argument");
        return GSI_ERR_INVALID_ARG;
    }
    *s = r->stats;
    return GSI_OK;
}

void gsi_result_free(gsi_result *r) {
    if (!r) return;
    cudaSetDevice(r->device);
    delete r;
}

gsi_status gsi_debug_lookup(const gsi_graph *g, int64_t nq, const int32_t *v, const int32_t *l, int64_t *len,
                            int32_t *groups_read, int32_t *nbrs, int64_t cap) {
    if (!g || nq < 0 || (nq && (!v || !l))) {
        set_error("invalid argument");
        return GSI_ERR_INVALID_ARG;
    }
    GSI_TRY(need_device());
    return debug_lookup_impl(g, nq, v, l, len, groups_read, nbrs, cap);
}

gsi_status gsi_debug_signatures(const gsi_graph *g, uint32_t *planes) {
    if (!g || !planes) {
        set_error("null argument");
        return GSI_ERR_INVALID_ARG;
    }
    GSI_TRY(need_device());
    GSI_CUDA(cudaSetDevice(g->device));
    if (g->n) GSI_CUDA(cudaMemcpy(planes, g->sig, 4ull * kPlanes * g->n, cudaMemcpyDeviceToHost));
    return GSI_OK;
}

gsi_status gsi_debug_filter(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                            const int32_t *qd, const int32_t *qe, int32_t mode, uint32_t *bitmaps, int64_t *counts) {
    GSI_TRY(need_device());
    return debug_filter_impl(g, k, qvl, qm, qs, qd, qe, mode, bitmaps, counts);
}

gsi_status gsi_debug_query_signatures(int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs, const int32_t *qd,
                                      const int32_t *qe, int32_t distinct, uint32_t *qsig) {
    if (k < 1 || k > GSI_MAX_K || !qvl || !qsig || (qm && (!qs || !qd || !qe))) {
        set_error("invalid argument");
        return GSI_ERR_INVALID_ARG;
    }
    encode_query_signatures(k, qvl, qm, qs, qd, qe, qsig, distinct ? 1 : 0);
    return GSI_OK;
}

const char *gsi_last_error(void) { return g_last_error.c_str(); }

const char *gsi_version(void) { return "gsi-b200 0.1 (sm_100a)"; }

int32_t gsi_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

}  // extern "C"
