// Internal structures of the C-ABI library (not part of the ABI).
// PAPER.md citations as "P:n" (/root/reference/PAPER.md line n).
#pragma once

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: no-ops unless a profiler tool is attached

#include "rpq.h"

// NVTX range over a C-ABI call (nsys / ncu --nvtx timelines)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// ---- error reporting (thread-local message, rpq_last_error) --------------
rpq_status rpq_fail(rpq_status st, const char *fmt, ...);
void rpq_clear_error();

// ---- graph: per-label CSR ("a separate grid for each edge label") --
struct LabelCSR {
    uint32_t *off = nullptr;     // device [nv + 1]
    uint32_t *nbr = nullptr;     // device [m], ascending per row
    uint64_t m = 0;              // distinct edges with this label
    uint32_t src_min = 1, src_max = 0;   // empty label: min > max
    uint32_t dst_min = 1, dst_max = 0;
    uint32_t max_deg = 0;        // largest row (long rows go to the hub kernel)
};

struct rpq_graph {
    int device = 0;
    uint32_t nv = 0;
    uint64_t ne = 0;             // distinct (u,l,w) triples (reading R4)
    std::vector<std::string> label_names;
    std::vector<std::string> vlabel_names;
    std::vector<LabelCSR> csr;   // [num_labels]
    std::vector<LabelCSR> in_csr;   // [num_labels] in-edges (RPQ_GRAPH_IN_EDGES), else empty
    uint32_t *off_base[2] = {nullptr, nullptr};   // [out/in] all labels' offsets (one block)
    uint32_t *nbr_base[2] = {nullptr, nullptr};   // [out/in] all labels' neighbours (one block)
    uint16_t *vlabel = nullptr;  // device [nv] or null
    std::vector<uint16_t> h_vlabel;   // host copy (CRPQ planning)
    // per label: is the edge set symmetric ((u,l,w) in E <=> (w,l,u) in E)?
    // -1 = not checked yet; filled lazily by label_symmetric (eval.cu)
    mutable std::mutex sym_mu;
    mutable std::vector<int8_t> sym;
    // allocator the CSR blocks came from (rpq_set_allocator at load time;
    // null functions = cudaMalloc / cudaFree)
    struct AllocSnap *alloc_snap = nullptr;
    // Per-graph query-plan cache (the graph is immutable, so these depend
    // only on the automaton): all-pairs candidates 0..nv-1, the productive
    // sources of each set of labels leaving q0 (device + host copies), and
    // the sparse/dense engine decision per automaton.  Filled by the first
    // all-pairs query that needs them; freed with the graph.
    struct ProdEntry {
        uint32_t reverse;
        std::vector<uint32_t> labels;    // sorted labels of q0's transitions
        uint32_t *d_pidx = nullptr;      // productive candidate indices (graph-owned)
        std::vector<uint32_t> h_pidx;
    };
    mutable std::mutex plan_mu;
    mutable uint32_t *d_iota = nullptr;  // [nv] 0, 1, ..., nv - 1
    mutable std::vector<ProdEntry *> prod_cache;
    mutable std::vector<std::pair<std::vector<uint32_t>, int>> engine_cache;   // automaton signature -> sparse?
    // CSR blocks of labels added after load (rpq_graph_add_label)
    std::vector<void *> extra_blocks;
};
// graph-owned device blocks (rpq_set_allocator at load time, else cudaMalloc)
void *graph_alloc(const rpq_graph *g, size_t bytes, void *stream);
void graph_block_free(const rpq_graph *g, void *p);

// ---- automaton ("automata plan") ------------------------------
struct rpq_nfa {
    uint32_t nq = 0;                 // states; 0 is initial
    uint64_t final_mask = 0;         // bit q set => q final
    bool accepts_empty = false;      // initial state final (epsilon in L)
    bool is_dfa = true;
    std::vector<uint32_t> from, label, to;   // sorted by (from, label, to)
    std::vector<uint32_t> off;       // [nq + 1] transitions of state q: off[q]..off[q+1]
    uint32_t vocab_size = 0;
    std::vector<std::string> vocab;  // label names the ids refer to
};

// ---- result --------------------------------------------------------------
struct rpq_result {
    int device = 0;
    uint32_t ncols = 0;
    uint64_t nrows = 0;              // rows materialised (PAIRS / CRPQ)
    uint32_t *cols[RPQ_MAX_COLS] = {};   // device column buffers
    uint64_t count = 0;              // result size (also in COUNT-only mode)
    // RPQ_PER_SOURCE: non-zero (source, count), ascending source (device)
    uint32_t *ps_src = nullptr;
    uint64_t *ps_cnt = nullptr;
    uint64_t *ps_pe = nullptr;       // RPQ_SOURCE_PE: product edges per listed source (PE, reading R12)
    uint64_t n_ps = 0;
    rpq_stats stats{};
    // PAIRS / PER_SOURCE: this shard's batches in evaluation order (rows of
    // batch k are [offset, offset + count) of the result)
    std::vector<rpq_batch_info> batches;
    // buffers are freed on the stream they were allocated on, through the
    // allocator that was installed when they were allocated
    void *stream = nullptr;
    struct AllocSnap *alloc_snap = nullptr;
};

// ---- device memory (stream-ordered pool allocator) -----------------------
void *dev_alloc(size_t bytes, void *stream);          // nullptr on failure
void dev_free(void *p, void *stream);
// the allocator installed right now (rpq_set_allocator), captured by objects
// that outlive a call; freed with the same functions later
struct AllocSnap {
    void *(*alloc)(size_t, void *, void *) = nullptr;
    void (*free_)(void *, void *, void *) = nullptr;
    void *ctx = nullptr;
};
AllocSnap *alloc_snapshot();                          // new'd copy of the current allocator
void dev_free_snap(void *p, void *stream, const AllocSnap *snap);
template <class T>
inline bool dev_alloc_to(T *&p, size_t bytes, void *stream) {
    p = static_cast<T *>(dev_alloc(bytes, stream));
    return p != nullptr;
}
uint64_t dev_available(bool *cached = nullptr);       // free + pool-reserved-unused bytes (cached)
void dev_available_invalidate();
void rpq_result_release(rpq_result *r);

// ---- evaluation driver (eval.cu) -----------------------------------------
// sources: device, sorted ascending, distinct, < nv (nullptr => all of V)
rpq_status eval_sources_device(const rpq_graph *g, const rpq_nfa *a, const uint32_t *d_sources,
                               uint64_t nsrc, const rpq_eval_opts *opts, rpq_result **out);

// ---- batch plan (plan.cpp) -----------------------------------------------
// jstart[b] = first candidate index owned by batch b (nb_eff + 1 entries)
void batch_plan(const uint32_t *bfirst, uint64_t nbatches, uint64_t nsrc, std::vector<uint64_t> &jstart);

// ---- compile (regex.cpp) -------------------------------------------------
rpq_status compile_regex(const std::vector<std::string> &vocab, const char *regex, uint32_t flags,
                         rpq_nfa **out, size_t *err_offset);
rpq_status reverse_automaton(const rpq_nfa *a, rpq_nfa **out);

#define RPQ_CUDA_TRY(expr)                                                              \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return rpq_fail(_e == cudaErrorMemoryAllocation ? RPQ_ENOMEM : RPQ_ECUDA,  \
                            "%s:%d %s: %s", __FILE__, __LINE__, #expr,                  \
                            cudaGetErrorString(_e));                                    \
    } while (0)
