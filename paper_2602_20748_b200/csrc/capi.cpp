// C-ABI plumbing: errors, automaton queries, result accessors, allocator.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstring>
#include <chrono>
#include <mutex>

#include "internal.h"

static thread_local std::string g_last_error;

rpq_status rpq_fail(rpq_status st, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

void rpq_clear_error() { g_last_error.clear(); }

extern "C" const char *rpq_last_error(void) { return g_last_error.c_str(); }

extern "C" const char *rpq_version(void) {
    return "rpq-b200 0.1 (sm_100a; per-label CSR; bit-parallel multi-source product BFS)";
}

extern "C" rpq_status rpq_device_count(int *n) {
    if (!n) return rpq_fail(RPQ_EINVAL, "NULL");
    *n = 0;
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) { *n = 0; cudaGetLastError(); }
    return RPQ_OK;
}

// ---- stream-ordered device allocation -----------------------------------
// cudaMallocAsync from the device's default pool with an unbounded release
// threshold: freed blocks stay reserved, so the per-query state arrays are
// recycled without cudaMalloc/cudaFree page-mapping costs.
static std::once_flag g_pool_once[64];

// optional caller allocator (rpq_set_allocator), e.g. a framework's caching
// allocator; replaces the pool for every device allocation of the library
namespace {
struct UserAlloc {
    void *(*alloc)(size_t, void *, void *) = nullptr;
    void (*free_)(void *, void *, void *) = nullptr;
    void *ctx = nullptr;
};
std::mutex g_ua_mu;
UserAlloc g_ua;
UserAlloc user_alloc() {
    std::lock_guard<std::mutex> lk(g_ua_mu);
    return g_ua;
}
}  // namespace

extern "C" rpq_status rpq_set_allocator(void *(*alloc)(size_t bytes, void *stream, void *ctx),
                                        void (*free_)(void *ptr, void *stream, void *ctx), void *ctx) {
    if ((alloc == nullptr) != (free_ == nullptr))
        return rpq_fail(RPQ_EINVAL, "rpq_set_allocator: give both functions or neither");
    std::lock_guard<std::mutex> lk(g_ua_mu);
    g_ua.alloc = alloc;
    g_ua.free_ = free_;
    g_ua.ctx = ctx;
    return RPQ_OK;
}

void *dev_alloc(size_t bytes, void *stream) {
    if (bytes == 0) bytes = 16;
    const UserAlloc ua = user_alloc();
    if (ua.alloc) return ua.alloc(bytes, stream, ua.ctx);
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(g_pool_once[dev & 63], [dev]() {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
    void *p = nullptr;
    if (cudaMallocAsync(&p, bytes, (cudaStream_t)stream) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

// Bytes an evaluation can still allocate: free device memory plus what the
// stream-ordered pool has reserved but is not using (it keeps freed blocks).
// cudaMemGetInfo is a driver (RM) call that was measured to stall for up to
// ~90 ms on the B200 boxes, so the value is cached per device; it is
// refreshed after 30 s, by graph load/free, and by an evaluation that ran out
// of memory under a cached budget (eval_sources_device retries once).
namespace {
struct MemCache {
    std::mutex m;
    bool valid = false;
    uint64_t bytes = 0;
    std::chrono::steady_clock::time_point t;
};
MemCache g_memcache[64];
}  // namespace

uint64_t dev_available(bool *cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    MemCache &c = g_memcache[dev & 63];
    std::lock_guard<std::mutex> lk(c.m);
    const auto now = std::chrono::steady_clock::now();
    if (c.valid && now - c.t < std::chrono::seconds(30)) {
        if (cached) *cached = true;
        return c.bytes;
    }
    if (cached) *cached = false;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) { cudaGetLastError(); return 0; }
    cudaMemPool_t pool;
    uint64_t reserved = 0, used = 0;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    }
    c.bytes = (uint64_t)free_b + (reserved > used ? reserved - used : 0);
    c.t = now;
    c.valid = true;
    return c.bytes;
}

void dev_available_invalidate() {
    for (MemCache &c : g_memcache) {
        std::lock_guard<std::mutex> lk(c.m);
        c.valid = false;
    }
}

extern "C" rpq_status rpq_trim_memory(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return rpq_fail(RPQ_EINVAL, "rpq_trim_memory: no CUDA device %d", device);
    }
    cudaMemPool_t pool;
    RPQ_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
    RPQ_CUDA_TRY(cudaDeviceSynchronize());
    RPQ_CUDA_TRY(cudaMemPoolTrimTo(pool, 0));
    dev_available_invalidate();
    return RPQ_OK;
}

void dev_free(void *p, void *stream) {
    if (!p) return;
    const UserAlloc ua = user_alloc();
    if (ua.free_) ua.free_(p, stream, ua.ctx);
    else cudaFreeAsync(p, (cudaStream_t)stream);
}

AllocSnap *alloc_snapshot() {
    const UserAlloc ua = user_alloc();
    AllocSnap *s = new AllocSnap();
    s->alloc = ua.alloc;
    s->free_ = ua.free_;
    s->ctx = ua.ctx;
    return s;
}

// free with the allocator captured when the block was allocated (not the
// one installed now); no snapshot = the current one
void dev_free_snap(void *p, void *stream, const AllocSnap *snap) {
    if (!p) return;
    if (!snap) { dev_free(p, stream); return; }
    if (snap->free_) snap->free_(p, stream, snap->ctx);
    else cudaFreeAsync(p, (cudaStream_t)stream);
}

// ---- automaton -----------------------------------------------------------
extern "C" rpq_status rpq_compile(const rpq_graph *vocab, const char *regex, uint32_t flags,
                                  rpq_nfa **out, size_t *err_offset) {
    if (out) *out = nullptr;
    if (!vocab) return rpq_fail(RPQ_EINVAL, "rpq_compile: NULL graph");
    return compile_regex(vocab->label_names, regex, flags, out, err_offset);
}

extern "C" rpq_status rpq_compile_labels(const char *const *names, uint32_t n, const char *regex,
                                         uint32_t flags, rpq_nfa **out, size_t *err_offset) {
    if (out) *out = nullptr;
    if (n && !names) return rpq_fail(RPQ_EINVAL, "rpq_compile_labels: NULL names");
    std::vector<std::string> v;
    for (uint32_t i = 0; i < n; ++i) v.emplace_back(names[i] ? names[i] : "");
    return compile_regex(v, regex, flags, out, err_offset);
}

extern "C" void rpq_nfa_free(rpq_nfa *a) { delete a; }

extern "C" rpq_status rpq_nfa_info(const rpq_nfa *a, uint32_t *nq, uint32_t *nt, uint32_t *nf,
                                   int *acc_empty, int *is_dfa) {
    if (!a) return rpq_fail(RPQ_EINVAL, "NULL automaton");
    if (nq) *nq = a->nq;
    if (nt) *nt = (uint32_t)a->from.size();
    if (nf) *nf = (uint32_t)__builtin_popcountll(a->final_mask);
    if (acc_empty) *acc_empty = a->accepts_empty;
    if (is_dfa) *is_dfa = a->is_dfa;
    return RPQ_OK;
}

extern "C" rpq_status rpq_nfa_transitions(const rpq_nfa *a, uint32_t *from, uint32_t *label,
                                          uint32_t *to, uint32_t cap, uint32_t *n,
                                          uint64_t *final_mask) {
    if (!a) return rpq_fail(RPQ_EINVAL, "NULL automaton");
    uint32_t cnt = (uint32_t)a->from.size();
    if (n) *n = cnt;
    if (final_mask) *final_mask = a->final_mask;
    if (cap < cnt) return cap == 0 && !from ? RPQ_OK : rpq_fail(RPQ_ECAPACITY, "need %u", cnt);
    for (uint32_t i = 0; i < cnt; ++i) {
        if (from) from[i] = a->from[i];
        if (label) label[i] = a->label[i];
        if (to) to[i] = a->to[i];
    }
    return RPQ_OK;
}

extern "C" rpq_status rpq_nfa_reverse(const rpq_nfa *a, rpq_nfa **out) {
    return reverse_automaton(a, out);
}

extern "C" rpq_status rpq_nfa_accepts(const rpq_nfa *a, const uint32_t *word, uint32_t len,
                                      int *accepted) {
    if (!a || !accepted || (len && !word)) return rpq_fail(RPQ_EINVAL, "NULL argument");
    uint64_t cur = a->nq ? 1ull : 0ull;
    for (uint32_t i = 0; i < len && cur; ++i) {
        uint64_t nxt = 0;
        for (uint32_t q = 0; q < a->nq; ++q) if ((cur >> q) & 1)
            for (uint32_t t = a->off[q]; t < a->off[q + 1]; ++t)
                if (a->label[t] == word[i]) nxt |= 1ull << a->to[t];
        cur = nxt;
    }
    *accepted = (cur & a->final_mask) != 0;
    return RPQ_OK;
}

// ---- results -------------------------------------------------------------
void rpq_result_release(rpq_result *r) {
    if (!r) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(r->device);
    // result buffers come from dev_alloc on the evaluation's stream: freed
    // on that stream (ordered after the caller's work queued there) through
    // the allocator that allocated them
    for (uint32_t c = 0; c < RPQ_MAX_COLS; ++c) if (r->cols[c]) dev_free_snap(r->cols[c], r->stream, r->alloc_snap);
    if (r->ps_src) dev_free_snap(r->ps_src, r->stream, r->alloc_snap);
    if (r->ps_cnt) dev_free_snap(r->ps_cnt, r->stream, r->alloc_snap);
    if (r->ps_pe) dev_free_snap(r->ps_pe, r->stream, r->alloc_snap);
    cudaSetDevice(prev);
    delete r->alloc_snap;
    delete r;
}

extern "C" void rpq_result_free(rpq_result *r) { rpq_result_release(r); }

extern "C" uint64_t rpq_result_count(const rpq_result *r) { return r ? r->count : 0; }

extern "C" rpq_status rpq_result_device_view(const rpq_result *r, const uint32_t **cols,
                                             uint32_t *ncols, uint64_t *n) {
    if (!r) return rpq_fail(RPQ_EINVAL, "NULL result");
    if (ncols) *ncols = r->ncols;
    if (n) *n = r->nrows;
    if (cols) for (uint32_t c = 0; c < r->ncols; ++c) cols[c] = r->cols[c];
    return RPQ_OK;
}

extern "C" rpq_status rpq_result_copy_host(const rpq_result *r, uint32_t *const *cols, uint64_t cap,
                                           uint64_t *n) {
    if (!r) return rpq_fail(RPQ_EINVAL, "NULL result");
    if (n) *n = r->nrows;
    if (cap < r->nrows) return rpq_fail(RPQ_ECAPACITY, "need %llu rows", (unsigned long long)r->nrows);
    if (!cols && r->nrows) return rpq_fail(RPQ_EINVAL, "NULL columns");
    cudaSetDevice(r->device);
    for (uint32_t c = 0; c < r->ncols; ++c)
        if (r->nrows) RPQ_CUDA_TRY(cudaMemcpy(cols[c], r->cols[c], r->nrows * 4, cudaMemcpyDeviceToHost));
    return RPQ_OK;
}

extern "C" rpq_status rpq_result_source_counts(const rpq_result *r, uint32_t *srcs, uint64_t *counts,
                                               uint64_t cap, uint64_t *n) {
    if (!r) return rpq_fail(RPQ_EINVAL, "NULL result");
    if (n) *n = r->n_ps;
    if (cap < r->n_ps) return rpq_fail(RPQ_ECAPACITY, "need %llu", (unsigned long long)r->n_ps);
    cudaSetDevice(r->device);
    if (r->n_ps) {
        if (srcs) RPQ_CUDA_TRY(cudaMemcpy(srcs, r->ps_src, r->n_ps * 4, cudaMemcpyDeviceToHost));
        if (counts) RPQ_CUDA_TRY(cudaMemcpy(counts, r->ps_cnt, r->n_ps * 8, cudaMemcpyDeviceToHost));
    }
    return RPQ_OK;
}

extern "C" rpq_status rpq_result_batches(const rpq_result *r, rpq_batch_info *out, uint64_t cap, uint64_t *n) {
    if (!r) return rpq_fail(RPQ_EINVAL, "NULL result");
    if (n) *n = r->batches.size();
    if (cap < r->batches.size()) return rpq_fail(RPQ_ECAPACITY, "need %zu", r->batches.size());
    if (!out && !r->batches.empty()) return rpq_fail(RPQ_EINVAL, "NULL output");
    for (size_t i = 0; i < r->batches.size(); ++i) out[i] = r->batches[i];
    return RPQ_OK;
}

extern "C" rpq_status rpq_result_source_pe(const rpq_result *r, uint64_t *pe, uint64_t cap, uint64_t *n) {
    if (!r) return rpq_fail(RPQ_EINVAL, "NULL result");
    if (n) *n = r->ps_pe ? r->n_ps : 0;
    if (!r->ps_pe) return rpq_fail(RPQ_EINVAL, "result was not evaluated with RPQ_PER_SOURCE | RPQ_SOURCE_PE");
    if (cap < r->n_ps) return rpq_fail(RPQ_ECAPACITY, "need %llu", (unsigned long long)r->n_ps);
    cudaSetDevice(r->device);
    if (r->n_ps && pe) RPQ_CUDA_TRY(cudaMemcpy(pe, r->ps_pe, r->n_ps * 8, cudaMemcpyDeviceToHost));
    return RPQ_OK;
}

extern "C" rpq_status rpq_result_stats(const rpq_result *r, rpq_stats *s) {
    if (!r || !s) return rpq_fail(RPQ_EINVAL, "NULL argument");
    *s = r->stats;
    s->count = r->count;
    return RPQ_OK;
}
