// crpq_eval: conjunctive RPQs (Definition 2).
//
// A CRPQ is answered by "evaluating each RPQ atom and then combining the
// results using joins".  Here:
//   1. plan: order the atoms so that each one after the first shares a
//      variable with the bound set (atoms with a constant endpoint first);
//      a variable in no atom or a disconnected pattern is rejected
//      (EUNSUPPORTED, reading R18);
//   2. each atom x -rho-> y is evaluated by the RPQ kernels from the sources
//      its x can take: the distinct values already bound to x, else the
//      candidates of x (constant / vertex label condition (1) / all of V);
//      its pairs are filtered by y's candidates (and s == d when x == y);
//   3. the relation is joined with the table of bound tuples on the device:
//      expansion by binary search over the (src,dst)-sorted relation when
//      one endpoint is bound (the relation is re-sorted by (dst,src) when only
//      y is), semi-join when both are;
//   4. distinct-vertex filters, then a stable LSD radix sort gives
//      tuples in lexicographic variable order.  Tuples are distinct because
//      every relation is a set and each join step extends an assignment.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <vector>

#include "internal.h"

namespace {

struct VarPred {
    int64_t cst;               // -1 = free
    int32_t label;             // -1 = any
    const uint16_t *vlabel;
    __device__ __forceinline__ bool ok(uint32_t v) const {
        return (cst < 0 || (int64_t)v == cst) && (label < 0 || vlabel[v] == (uint16_t)label);
    }
};

inline int grid_for(uint64_t n, int block = 256) {
    uint64_t g = (n + block - 1) / block;
    if (g > 148ull * 16) g = 148ull * 16;
    return g ? (int)g : 1;
}

__global__ void k_cand_flags(VarPred p, uint32_t nv, uint8_t *flag) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x)
        flag[v] = p.ok((uint32_t)v);
}

__global__ void k_pair_flags(const uint32_t *src, const uint32_t *dst, uint64_t n, VarPred py, int same,
                             uint8_t *flag, VarPred px, int check_src) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        flag[i] = py.ok(dst[i]) && (!same || src[i] == dst[i]) && (!check_src || px.ok(src[i]));
}

__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t *a, uint64_t n, uint32_t key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// rows of the table joined with a relation sorted by key column `rk`
__global__ void k_join_count(const uint32_t *tkey, uint64_t nrows, const uint32_t *rk, uint64_t nrel,
                             unsigned long long *lo, unsigned long long *cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nrows; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = tkey[i];
        const uint64_t a = lower_bound_u32(rk, nrel, k);
        const uint64_t b = lower_bound_u32(rk, nrel, k + 1) ;
        lo[i] = a;
        cnt[i] = (k == 0xffffffffu) ? (nrel - a) : (b - a);
    }
}

__global__ void k_join_write(const uint32_t *const *tcols, uint32_t ncols, uint64_t nrows, const unsigned long long *lo,
                             const unsigned long long *cnt, const unsigned long long *off, const uint32_t *rval,
                             uint32_t *const *ocols) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nrows; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = cnt[i], o = off[i], l = lo[i];
        for (uint64_t k = 0; k < c; ++k) {
            for (uint32_t j = 0; j < ncols; ++j) ocols[j][o + k] = tcols[j][i];
            ocols[ncols][o + k] = rval[l + k];
        }
    }
}

// both endpoints bound: keep rows whose (x, y) is in the (src,dst)-sorted relation
__global__ void k_semijoin(const uint32_t *tx, const uint32_t *ty, uint64_t nrows, const uint32_t *rs,
                           const uint32_t *rd, uint64_t nrel, uint8_t *flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nrows; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = tx[i], y = ty[i];
        uint64_t a = lower_bound_u32(rs, nrel, x);
        uint64_t b = (x == 0xffffffffu) ? nrel : lower_bound_u32(rs, nrel, x + 1);
        while (a < b) {   // binary search of y in rd[a, b)
            const uint64_t mid = (a + b) >> 1;
            if (rd[mid] < y) a = mid + 1; else b = mid;
        }
        flag[i] = (a < nrel && rs[a] == x && rd[a] == y);
    }
}

__global__ void k_ne_flags(const uint32_t *a, const uint32_t *b, uint64_t n, uint8_t *flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        flag[i] = flag[i] && a[i] != b[i];
}

__global__ void k_pack_swap(const uint32_t *s, const uint32_t *d, uint64_t n, uint64_t *key) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        key[i] = ((uint64_t)d[i] << 32) | s[i];
}

__global__ void k_unpack(const uint64_t *key, uint64_t n, uint32_t *hi, uint32_t *lo) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        hi[i] = (uint32_t)(key[i] >> 32);
        lo[i] = (uint32_t)key[i];
    }
}

__global__ void k_gather(const uint32_t *in, const uint32_t *idx, uint64_t n, uint32_t *out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[idx[i]];
}

__global__ void k_iota32(uint32_t *x, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        x[i] = (uint32_t)i;
}

// ---- worst-case-optimal join (generic join, RPQ_WCOJ) --------------------
// One extension step of the variable-at-a-time join ("the WCOJ-based
// CQ method"; generic join / leapfrog intersection): every row of the table
// binds a prefix of the matching order; the candidates of the next variable
// are the INTERSECTION of the value lists of all atom indexes whose key end
// is already bound (index = the atom relation sorted by (key, value)), minus
// vertices failing the variable's label / constant, its self atoms (x -> x)
// and its distinct-vertex filters.  A warp per row: the smallest
// list is scanned by the lanes, every element binary-searched in the others.
constexpr int WJ_MAXC = 8;
struct ExtStep {
    int nc;                                    // constraining indexes
    const uint32_t *key[WJ_MAXC], *val[WJ_MAXC];
    uint64_t n[WJ_MAXC];
    int keycol[WJ_MAXC];                       // table column holding the index key
    int nd;                                    // distinct filters against bound columns
    int dcol[WJ_MAXC];
    VarPred pred;
    const uint8_t *selfok;                     // [nv] self atoms of the variable, or null
};

__device__ __forceinline__ bool in_sorted(const uint32_t *a, uint64_t lo, uint64_t hi, uint32_t x) {
    const uint64_t end = hi;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo < end && a[lo] == x;
}

// WRITE = false: cnt[row] = number of extensions; true: write them at off[row]
template <bool WRITE>
__global__ void k_wcoj_extend(const ExtStep st, const uint32_t *const *tcols, uint32_t ncols, uint64_t nrows,
                              unsigned long long *cnt, const unsigned long long *off, uint32_t *const *ocols) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (uint64_t r = wid; r < nrows; r += nwarps) {
        uint64_t lo[WJ_MAXC], hi[WJ_MAXC];
        int best = 0;
        for (int c = 0; c < st.nc; ++c) {   // equal range of the row's key in index c
            const uint32_t k = tcols[st.keycol[c]][r];
            lo[c] = lower_bound_u32(st.key[c], st.n[c], k);
            hi[c] = k == 0xffffffffu ? st.n[c] : lower_bound_u32(st.key[c], st.n[c], k + 1);
            if (hi[c] - lo[c] < hi[best] - lo[best]) best = c;
        }
        unsigned long long o = WRITE ? off[r] : 0ull, found = 0;
        for (uint64_t b0 = lo[best]; b0 < hi[best]; b0 += 32) {
            const uint64_t i = b0 + lane;
            bool ok = i < hi[best];
            uint32_t e = ok ? st.val[best][i] : 0u;
            ok = ok && st.pred.ok(e) && (!st.selfok || st.selfok[e]);
            for (int d = 0; d < st.nd && ok; ++d) ok = e != tcols[st.dcol[d]][r];
            for (int c = 0; c < st.nc && ok; ++c)
                if (c != best) ok = in_sorted(st.val[c], lo[c], hi[c], e);
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            if (WRITE && ok) {
                const unsigned long long p = o + found + __popc(m & lt);
                for (uint32_t j = 0; j < ncols; ++j) ocols[j][p] = tcols[j][r];
                ocols[ncols][p] = e;
            }
            found += __popc(m);
        }
        if (!WRITE && lane == 0) cnt[r] = found;
    }
}

__global__ void k_mark_keys(const uint32_t *key, uint64_t n, uint8_t *mark) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        mark[key[i]] = 1;
}

__global__ void k_and_flags(uint8_t *a, const uint8_t *b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = a[i] && b[i];
}

// self atom x -rho-> x: mark v with (v, v) in the relation
__global__ void k_mark_self(const uint32_t *s, const uint32_t *d, uint64_t n, uint8_t *mark) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (s[i] == d[i]) mark[s[i]] = 1;
}

// ---- host helpers ---------------------------------------------------------
struct Pool {
    cudaStream_t s;
    std::vector<void *> ptrs;
    ~Pool() { for (void *p : ptrs) dev_free(p, s); }
    void *get(size_t b) {
        void *p = dev_alloc(b ? b : 16, s);
        if (p) ptrs.push_back(p);
        return p;
    }
    void put(void *p) {
        auto it = std::find(ptrs.begin(), ptrs.end(), p);
        if (it != ptrs.end()) { dev_free(p, s); ptrs.erase(it); }
    }
};

struct Table {
    std::vector<uint32_t> vars;        // bound variables, column order
    std::vector<uint32_t *> cols;      // device columns (Pool-owned)
    uint64_t n = 0;
    int col_of(uint32_t v) const {
        for (size_t i = 0; i < vars.size(); ++i) if (vars[i] == v) return (int)i;
        return -1;
    }
};

// compact the columns of a table by a flag array
rpq_status compact(Pool &P, std::vector<uint32_t *> &cols, uint64_t &n, const uint8_t *flag, cudaStream_t s) {
    if (n == 0) return RPQ_OK;
    uint64_t *d_n = (uint64_t *)P.get(8);
    size_t tb = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, cols[0], flag, cols[0], d_n, (int64_t)n, s);
    void *tmp = P.get(tb);
    if (!d_n || !tmp) return rpq_fail(RPQ_ENOMEM, "crpq: out of device memory");
    uint64_t m = 0;
    for (auto &c : cols) {
        uint32_t *o = (uint32_t *)P.get(n * 4);
        if (!o) return rpq_fail(RPQ_ENOMEM, "crpq: out of device memory");
        cub::DeviceSelect::Flagged(tmp, tb, c, flag, o, d_n, (int64_t)n, s);
        P.put(c);
        c = o;
    }
    RPQ_CUDA_TRY(cudaMemcpyAsync(&m, d_n, 8, cudaMemcpyDeviceToHost, s));
    RPQ_CUDA_TRY(cudaStreamSynchronize(s));
    n = m;
    return RPQ_OK;
}

void add_stats(rpq_stats &a, const rpq_stats &b) {
    a.product_edges += b.product_edges;
    a.word_items += b.word_items;
    a.word_edge_ops += b.word_edge_ops;
    a.items += b.items;
    a.item_edges += b.item_edges;
    a.item_transitions += b.item_transitions;
    a.activations += b.activations;
    a.next_reds += b.next_reds;
    a.levels += b.levels;
    a.batches += b.batches;
    a.expand_launches += b.expand_launches;
    a.kernel_launches += b.kernel_launches;
    a.expand_ms += b.expand_ms;
}

// Generic join (RPQ_WCOJ): fills T with every variable bound (columns in the
// matching order), distinct filters applied during the extension steps.
rpq_status wcoj_join(const rpq_graph *g, const crpq_query *q, const rpq_eval_opts &o, cudaStream_t s, Pool &P,
                     rpq_stats &ST, const std::vector<int32_t> &vlab, const std::vector<int64_t> &vcst, Table &T) {
    const uint32_t nvars = q->num_vars, natoms = q->num_atoms;
    auto pred = [&](uint32_t v) { return VarPred{vcst[v], vlab[v], g->vlabel}; };
    // ---- matching order: a constant (else the most-constrained variable)
    // first, then repeatedly the variable with the most atoms into the bound
    // set (ties: constant / label, then lowest id); disconnected -> R18
    std::vector<int> pos(nvars, -1);
    std::vector<uint32_t> ord;
    for (uint32_t k = 0; k < nvars; ++k) {
        int best = -1;
        long bs = -1;
        for (uint32_t v = 0; v < nvars; ++v) {
            if (pos[v] >= 0) continue;
            long links = 0, deg = 0;
            for (uint32_t i = 0; i < natoms; ++i) {
                const uint32_t x = q->atom_x[i], y = q->atom_y[i];
                if (x != v && y != v) continue;
                ++deg;
                const uint32_t o2 = x == v ? y : x;
                if (o2 != v && pos[o2] >= 0) ++links;
            }
            if (k > 0 && links == 0) continue;
            const long sc = links * 10000 + (vcst[v] >= 0 ? 1000 : 0) + (vlab[v] >= 0 ? 100 : 0) + deg;
            if (sc > bs) { bs = sc; best = (int)v; }
        }
        if (best < 0) return rpq_fail(RPQ_EUNSUPPORTED, "crpq_eval: disconnected pattern (R18)");
        pos[best] = (int)k;
        ord.push_back((uint32_t)best);
    }
    // ---- atom indexes, keyed by the end bound first ----
    struct Index { uint32_t keyvar, valvar; uint32_t *key, *val; uint64_t n; };
    std::vector<Index> idx;
    std::vector<uint8_t *> selfok(nvars, nullptr);
    const bool in_edges = g->in_csr.size() == g->csr.size();
    for (uint32_t i = 0; i < natoms; ++i) {
        const uint32_t x = q->atom_x[i], y = q->atom_y[i];
        const bool self = x == y;
        const bool fwd = self || pos[x] < pos[y];
        const uint32_t kv = fwd ? x : y;           // key end = bound first
        // traverse from the key end: forward from x, or the reversed
        // automaton over the transposed graph from y (reverse plan);
        // without in-edges, forward from all x and re-sort by (y, x)
        const bool backward = !fwd && in_edges && !getenv("RPQ_CRPQ_FORWARD");
        const uint32_t sv = fwd || backward ? kv : x;
        rpq_nfa *rev = nullptr;
        struct RevGuard { rpq_nfa **p; ~RevGuard() { delete *p; } } rg0{&rev};
        if (backward) {
            rpq_status rs = reverse_automaton(q->atom_nfa[i], &rev);
            if (rs != RPQ_OK) return rs;
        }
        uint32_t *srcs = nullptr;
        uint64_t nsrc = 0;
        bool all_v = true;
        if (vcst[sv] >= 0 || vlab[sv] >= 0) {   // candidates of the start variable
            all_v = false;
            uint8_t *flag = (uint8_t *)P.get(g->nv);
            srcs = (uint32_t *)P.get((uint64_t)g->nv * 4);
            uint64_t *d_n = (uint64_t *)P.get(8);
            if (!flag || !srcs || !d_n) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            k_cand_flags<<<grid_for(g->nv), 256, 0, s>>>(pred(sv), g->nv, flag);
            size_t tb = 0;
            thrust::counting_iterator<uint32_t> it(0);
            cub::DeviceSelect::Flagged(nullptr, tb, it, flag, srcs, d_n, (int64_t)g->nv, s);
            void *tmp = P.get(tb);
            if (!tmp) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            cub::DeviceSelect::Flagged(tmp, tb, it, flag, srcs, d_n, (int64_t)g->nv, s);
            RPQ_CUDA_TRY(cudaMemcpyAsync(&nsrc, d_n, 8, cudaMemcpyDeviceToHost, s));
            RPQ_CUDA_TRY(cudaStreamSynchronize(s));
        }
        rpq_eval_opts ao = o;
        ao.mode = RPQ_PAIRS | (o.mode & (RPQ_STATS | RPQ_TIME_KERNELS));
        ao.shard_index = 0;
        ao.shard_count = 1;
        if (backward) ao.reserved |= 2u;
        rpq_result *rel = nullptr;
        const rpq_nfa *enfa = backward ? rev : q->atom_nfa[i];
        rpq_status st = all_v ? eval_sources_device(g, enfa, nullptr, 0, &ao, &rel)
                              : eval_sources_device(g, enfa, srcs, nsrc, &ao, &rel);
        if (st != RPQ_OK) return st;
        add_stats(ST, rel->stats);
        struct RelGuard { rpq_result *r; ~RelGuard() { rpq_result_release(r); } } rg{rel};
        uint64_t n = rel->nrows;
        // pool-owned (key, value) columns: forward and backward results are
        // already sorted by (key, value); forward-evaluated backward indexes
        // are re-sorted by (y, x)
        std::vector<uint32_t *> rc(2);
        for (int c = 0; c < 2; ++c) {
            rc[c] = (uint32_t *)P.get(std::max<uint64_t>(n, 1) * 4);
            if (!rc[c]) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            if (n) RPQ_CUDA_TRY(cudaMemcpyAsync(rc[c], rel->cols[c], n * 4, cudaMemcpyDeviceToDevice, s));
        }
        const uint32_t vv = self ? x : (fwd ? y : x);   // value end
        if (!fwd && !backward && n) {
            uint64_t *k1 = (uint64_t *)P.get(n * 8), *k2 = (uint64_t *)P.get(n * 8);
            if (!k1 || !k2) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            k_pack_swap<<<grid_for(n), 256, 0, s>>>(rc[0], rc[1], n, k1);
            size_t tb = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, tb, k1, k2, (int64_t)n, 0, 64, s);
            void *tmp = P.get(tb);
            if (!tmp) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            cub::DeviceRadixSort::SortKeys(tmp, tb, k1, k2, (int64_t)n, 0, 64, s);
            k_unpack<<<grid_for(n), 256, 0, s>>>(k2, n, rc[0], rc[1]);   // (y, x)
        }
        if (self) {   // x -rho-> x: a filter on x's candidates
            if (!selfok[x]) {
                selfok[x] = (uint8_t *)P.get(g->nv);
                if (!selfok[x]) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
                RPQ_CUDA_TRY(cudaMemsetAsync(selfok[x], 1, g->nv, s));
            }
            uint8_t *m = (uint8_t *)P.get(g->nv);
            if (!m) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            RPQ_CUDA_TRY(cudaMemsetAsync(m, 0, g->nv, s));
            if (n) k_mark_self<<<grid_for(n), 256, 0, s>>>(rc[0], rc[1], n, m);
            k_and_flags<<<grid_for(g->nv), 256, 0, s>>>(selfok[x], m, g->nv);
            continue;
        }
        // drop pairs whose value fails its variable's label / constant
        if (n) {
            uint8_t *flag = (uint8_t *)P.get(n);
            if (!flag) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            k_pair_flags<<<grid_for(n), 256, 0, s>>>(rc[0], rc[1], n, pred(vv), 0, flag, pred(kv), 1);
            st = compact(P, rc, n, flag, s);
            if (st != RPQ_OK) return st;
        }
        idx.push_back(Index{kv, vv, rc[0], rc[1], n});
    }
    // ---- first variable: its candidates that occur as a key of every index
    const uint32_t v0 = ord[0];
    {
        uint8_t *flag = (uint8_t *)P.get(g->nv), *m = (uint8_t *)P.get(g->nv);
        uint32_t *c0 = (uint32_t *)P.get((uint64_t)g->nv * 4);
        uint64_t *d_n = (uint64_t *)P.get(8);
        if (!flag || !m || !c0 || !d_n) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
        k_cand_flags<<<grid_for(g->nv), 256, 0, s>>>(pred(v0), g->nv, flag);
        if (selfok[v0]) k_and_flags<<<grid_for(g->nv), 256, 0, s>>>(flag, selfok[v0], g->nv);
        for (auto &ix : idx) {
            if (ix.keyvar != v0) continue;
            RPQ_CUDA_TRY(cudaMemsetAsync(m, 0, g->nv, s));
            if (ix.n) k_mark_keys<<<grid_for(ix.n), 256, 0, s>>>(ix.key, ix.n, m);
            k_and_flags<<<grid_for(g->nv), 256, 0, s>>>(flag, m, g->nv);
        }
        size_t tb = 0;
        thrust::counting_iterator<uint32_t> it(0);
        cub::DeviceSelect::Flagged(nullptr, tb, it, flag, c0, d_n, (int64_t)g->nv, s);
        void *tmp = P.get(tb);
        if (!tmp) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
        cub::DeviceSelect::Flagged(tmp, tb, it, flag, c0, d_n, (int64_t)g->nv, s);
        uint64_t n0 = 0;
        RPQ_CUDA_TRY(cudaMemcpyAsync(&n0, d_n, 8, cudaMemcpyDeviceToHost, s));
        RPQ_CUDA_TRY(cudaStreamSynchronize(s));
        T.vars = {v0};
        T.cols = {c0};
        T.n = n0;
    }
    // ---- extension steps ----
    for (uint32_t k = 1; k < nvars; ++k) {
        const uint32_t v = ord[k];
        ExtStep es{};
        for (auto &ix : idx) {
            if (ix.valvar != v || T.col_of(ix.keyvar) < 0) continue;
            if (es.nc == WJ_MAXC) return rpq_fail(RPQ_EUNSUPPORTED, "crpq_eval: > %d atoms into one variable", WJ_MAXC);
            es.key[es.nc] = ix.key;
            es.val[es.nc] = ix.val;
            es.n[es.nc] = ix.n;
            es.keycol[es.nc] = T.col_of(ix.keyvar);
            ++es.nc;
        }
        for (uint32_t d = 0; d < q->num_distinct; ++d) {
            const uint32_t a = q->distinct_pairs[2 * d], b = q->distinct_pairs[2 * d + 1];
            const uint32_t other = a == v ? b : (b == v ? a : UINT32_MAX);
            if (other == UINT32_MAX) continue;
            if (other == v) { T.n = 0; break; }            // distinct(v, v): nothing survives
            const int c = T.col_of(other);
            if (c < 0) continue;                            // filtered when `other` is bound
            if (es.nd == WJ_MAXC) return rpq_fail(RPQ_EUNSUPPORTED, "crpq_eval: too many distinct filters");
            es.dcol[es.nd++] = c;
        }
        es.pred = pred(v);
        es.selfok = selfok[v];
        uint32_t **d_in = (uint32_t **)P.get(T.cols.size() * sizeof(void *));
        unsigned long long *cnt = (unsigned long long *)P.get(std::max<uint64_t>(T.n, 1) * 8);
        unsigned long long *off = (unsigned long long *)P.get(std::max<uint64_t>(T.n, 1) * 8);
        if (!d_in || !cnt || !off) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
        RPQ_CUDA_TRY(cudaMemcpyAsync(d_in, T.cols.data(), T.cols.size() * sizeof(void *), cudaMemcpyHostToDevice, s));
        uint64_t total = 0;
        const int wg = grid_for(T.n * 32);
        if (T.n) {
            k_wcoj_extend<false><<<wg, 256, 0, s>>>(es, d_in, (uint32_t)T.cols.size(), T.n, cnt, nullptr, nullptr);
            size_t tb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int64_t)T.n, s);
            void *tmp = P.get(tb);
            if (!tmp) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int64_t)T.n, s);
            unsigned long long a = 0, b = 0;
            RPQ_CUDA_TRY(cudaMemcpyAsync(&a, off + T.n - 1, 8, cudaMemcpyDeviceToHost, s));
            RPQ_CUDA_TRY(cudaMemcpyAsync(&b, cnt + T.n - 1, 8, cudaMemcpyDeviceToHost, s));
            RPQ_CUDA_TRY(cudaStreamSynchronize(s));
            total = a + b;
        }
        std::vector<uint32_t *> nc(T.cols.size() + 1);
        for (auto &c : nc) {
            c = (uint32_t *)P.get(std::max<uint64_t>(total, 1) * 4);
            if (!c) return rpq_fail(RPQ_ENOMEM, "crpq: out of device memory (%llu tuples)", (unsigned long long)total);
        }
        if (total) {
            uint32_t **d_out = (uint32_t **)P.get(nc.size() * sizeof(void *));
            if (!d_out) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            RPQ_CUDA_TRY(cudaMemcpyAsync(d_out, nc.data(), nc.size() * sizeof(void *), cudaMemcpyHostToDevice, s));
            k_wcoj_extend<true><<<wg, 256, 0, s>>>(es, d_in, (uint32_t)T.cols.size(), T.n, cnt, off, d_out);
        }
        for (auto c : T.cols) P.put(c);
        T.cols = nc;
        T.vars.push_back(v);
        T.n = total;
    }
    return RPQ_OK;
}

}  // namespace

// rows differing from the previous one (rows sorted): the distinct projection
__global__ void k_row_changed(const uint32_t *const *cols, uint32_t ncols, uint64_t n, uint8_t *flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        bool d = i == 0;
        for (uint32_t c = 0; c < ncols && !d; ++c) d = cols[c][i] != cols[c][i - 1];
        flag[i] = d;
    }
}

static rpq_status crpq_impl(const rpq_graph *g, const crpq_query *q, const rpq_eval_opts *opts_in,
                            const std::vector<uint32_t> &outv, rpq_result **out);

extern "C" rpq_status crpq_eval(const rpq_graph *g, const crpq_query *q, const rpq_eval_opts *opts_in,
                                rpq_result **out) {
    NvtxRange nvtx_("crpq_eval");
    if (out) *out = nullptr;
    if (!g || !q || !out) return rpq_fail(RPQ_EINVAL, "crpq_eval: NULL argument");
    std::vector<uint32_t> all(q->num_vars);
    for (uint32_t v = 0; v < q->num_vars; ++v) all[v] = v;
    return crpq_impl(g, q, opts_in, all, out);
}

extern "C" rpq_status crpq_eval_project(const rpq_graph *g, const crpq_query *q, const uint32_t *out_vars,
                                        uint32_t num_out, const rpq_eval_opts *opts_in, rpq_result **out) {
    NvtxRange nvtx_("crpq_eval_project");
    if (out) *out = nullptr;
    if (!g || !q || !out || !out_vars || num_out == 0) return rpq_fail(RPQ_EINVAL, "crpq_eval_project: bad argument");
    std::vector<uint32_t> ov(out_vars, out_vars + num_out);
    for (uint32_t i = 0; i < num_out; ++i) {
        if (ov[i] >= q->num_vars) return rpq_fail(RPQ_EINVAL, "crpq_eval_project: output variable %u", ov[i]);
        for (uint32_t j = 0; j < i; ++j)
            if (ov[j] == ov[i]) return rpq_fail(RPQ_EINVAL, "crpq_eval_project: repeated output variable");
    }
    return crpq_impl(g, q, opts_in, ov, out);
}

static rpq_status crpq_impl(const rpq_graph *g, const crpq_query *q, const rpq_eval_opts *opts_in,
                            const std::vector<uint32_t> &outv, rpq_result **out) {
    const uint32_t nvars = q->num_vars, natoms = q->num_atoms;
    if (nvars == 0 || nvars > RPQ_MAX_COLS) return rpq_fail(RPQ_EINVAL, "crpq_eval: 1..%d variables", RPQ_MAX_COLS);
    if (natoms == 0 || !q->atom_x || !q->atom_y || !q->atom_nfa)
        return rpq_fail(RPQ_EINVAL, "crpq_eval: no atoms");
    std::vector<int32_t> vlab(nvars, -1);
    std::vector<int64_t> vcst(nvars, -1);
    for (uint32_t v = 0; v < nvars; ++v) {
        if (q->var_label) vlab[v] = q->var_label[v];
        if (q->var_const) vcst[v] = q->var_const[v];
        if (vlab[v] >= 65536 || (vlab[v] >= 0 && !g->vlabel))
            return rpq_fail(RPQ_EINVAL, "crpq_eval: variable %u has a vertex label but the graph has none", v);
        if (vcst[v] >= (int64_t)g->nv) return rpq_fail(RPQ_EINVAL, "crpq_eval: constant >= |V|");
    }
    std::vector<int> used(nvars, 0);
    for (uint32_t i = 0; i < natoms; ++i) {
        if (q->atom_x[i] >= nvars || q->atom_y[i] >= nvars || !q->atom_nfa[i])
            return rpq_fail(RPQ_EINVAL, "crpq_eval: bad atom %u", i);
        used[q->atom_x[i]] = used[q->atom_y[i]] = 1;
    }
    for (uint32_t v = 0; v < nvars; ++v)
        if (!used[v]) return rpq_fail(RPQ_EUNSUPPORTED, "crpq_eval: variable %u occurs in no atom (R18)", v);
    for (uint32_t i = 0; i < q->num_distinct; ++i)
        if (!q->distinct_pairs || q->distinct_pairs[2 * i] >= nvars || q->distinct_pairs[2 * i + 1] >= nvars)
            return rpq_fail(RPQ_EINVAL, "crpq_eval: bad distinct filter");

    rpq_eval_opts o{};
    if (opts_in) o = *opts_in;
    const bool wcoj = (o.mode & RPQ_WCOJ) != 0;

    // ---- plan: constants first, then atoms sharing a bound variable -------
    std::vector<uint32_t> order;
    std::vector<int> done(natoms, 0), bound(nvars, 0);
    auto score = [&](uint32_t i) {
        const uint32_t x = q->atom_x[i], y = q->atom_y[i];
        int s = 0;
        if (vcst[x] >= 0 || vcst[y] >= 0) s += 8;
        if (bound[x]) s += 4;
        if (bound[y]) s += 2;
        if (vlab[x] >= 0) s += 1;
        return s;
    };
    for (uint32_t k = 0; k < natoms; ++k) {
        int best = -1, bs = -1;
        for (uint32_t i = 0; i < natoms; ++i) {
            if (done[i]) continue;
            const bool connected = k == 0 || bound[q->atom_x[i]] || bound[q->atom_y[i]];
            if (!connected) continue;
            const int sc = score(i);
            if (sc > bs) { bs = sc; best = (int)i; }
        }
        if (best < 0) return rpq_fail(RPQ_EUNSUPPORTED, "crpq_eval: disconnected pattern (R18)");
        done[best] = 1;
        bound[q->atom_x[best]] = bound[q->atom_y[best]] = 1;
        order.push_back((uint32_t)best);
    }

    RPQ_CUDA_TRY(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)o.cuda_stream;
    Pool P{s, {}};
    rpq_stats ST{};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    auto pred = [&](uint32_t v) { return VarPred{vcst[v], vlab[v], g->vlabel}; };

    Table T;
    if (wcoj) {
        rpq_status wst = wcoj_join(g, q, o, s, P, ST, vlab, vcst, T);
        if (wst != RPQ_OK) return wst;
    }
    for (uint32_t k = 0; k < (wcoj ? 0u : natoms); ++k) {
        const uint32_t ai = order[k];
        const uint32_t x = q->atom_x[ai], y = q->atom_y[ai];
        const rpq_nfa *nfa = q->atom_nfa[ai];
        const int cx = T.col_of(x), cy = T.col_of(y);
        // ---- sources of the atom ----
        // Backward (reverse plan): x free and unconstrained by a
        // constant, y bound or constant, in-edges loaded -> evaluate the
        // reversed automaton over the transposed graph from y's values; the
        // relation then comes sorted by (y, x).
        const bool backward = cx < 0 && vcst[x] < 0 && (cy >= 0 || vcst[y] >= 0) &&
                              g->in_csr.size() == g->csr.size() && !getenv("RPQ_CRPQ_FORWARD");
        const uint32_t sv = backward ? y : x;      // the side the traversal starts from
        const int csv = backward ? cy : cx;
        rpq_nfa *rev_nfa = nullptr;
        struct RevGuard { rpq_nfa **p; ~RevGuard() { delete *p; } } revg{&rev_nfa};
        if (backward) {
            rpq_status rs = reverse_automaton(nfa, &rev_nfa);
            if (rs != RPQ_OK) return rs;
        }
        uint32_t *srcs = nullptr;
        uint64_t nsrc = 0;
        bool all_v = false;
        if (csv >= 0) {
            // distinct values bound to x
            uint32_t *tmpk = (uint32_t *)P.get(T.n * 4), *sorted = (uint32_t *)P.get(T.n * 4);
            srcs = (uint32_t *)P.get(T.n * 4);
            uint64_t *d_n = (uint64_t *)P.get(8);
            if (!tmpk || !sorted || !srcs || !d_n) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            RPQ_CUDA_TRY(cudaMemcpyAsync(tmpk, T.cols[csv], T.n * 4, cudaMemcpyDeviceToDevice, s));
            size_t t1 = 0, t2 = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, t1, tmpk, sorted, (int64_t)T.n, 0, 32, s);
            cub::DeviceSelect::Unique(nullptr, t2, sorted, srcs, d_n, (int64_t)T.n, s);
            void *tmp = P.get(std::max(t1, t2));
            if (!tmp) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            cub::DeviceRadixSort::SortKeys(tmp, t1, tmpk, sorted, (int64_t)T.n, 0, 32, s);
            cub::DeviceSelect::Unique(tmp, t2, sorted, srcs, d_n, (int64_t)T.n, s);
            RPQ_CUDA_TRY(cudaMemcpyAsync(&nsrc, d_n, 8, cudaMemcpyDeviceToHost, s));
            RPQ_CUDA_TRY(cudaStreamSynchronize(s));
        } else if (vcst[sv] >= 0) {
            srcs = (uint32_t *)P.get(4);
            if (!srcs) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            const uint32_t c = (uint32_t)vcst[sv];
            RPQ_CUDA_TRY(cudaMemcpyAsync(srcs, &c, 4, cudaMemcpyHostToDevice, s));
            RPQ_CUDA_TRY(cudaStreamSynchronize(s));
            nsrc = 1;
        } else if (vlab[sv] >= 0) {
            uint8_t *flag = (uint8_t *)P.get(g->nv);
            srcs = (uint32_t *)P.get((uint64_t)g->nv * 4);
            uint64_t *d_n = (uint64_t *)P.get(8);
            if (!flag || !srcs || !d_n) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            k_cand_flags<<<grid_for(g->nv), 256, 0, s>>>(pred(sv), g->nv, flag);
            size_t tb = 0;
            thrust::counting_iterator<uint32_t> it(0);
            cub::DeviceSelect::Flagged(nullptr, tb, it, flag, srcs, d_n, (int64_t)g->nv, s);
            void *tmp = P.get(tb);
            if (!tmp) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            cub::DeviceSelect::Flagged(tmp, tb, it, flag, srcs, d_n, (int64_t)g->nv, s);
            RPQ_CUDA_TRY(cudaMemcpyAsync(&nsrc, d_n, 8, cudaMemcpyDeviceToHost, s));
            RPQ_CUDA_TRY(cudaStreamSynchronize(s));
        } else {
            all_v = true;
        }
        // ---- evaluate the atom (sorted distinct pairs) ----
        rpq_eval_opts ao = o;
        ao.mode = RPQ_PAIRS | (o.mode & (RPQ_STATS | RPQ_TIME_KERNELS));
        ao.shard_index = 0;
        ao.shard_count = 1;
        if (backward) ao.reserved |= 2u;           // in-edge CSR (transposed graph)
        const rpq_nfa *enfa = backward ? rev_nfa : nfa;
        rpq_result *rel = nullptr;
        rpq_status st = all_v ? eval_sources_device(g, enfa, nullptr, 0, &ao, &rel)
                              : eval_sources_device(g, enfa, srcs, nsrc, &ao, &rel);
        if (st != RPQ_OK) return st;
        add_stats(ST, rel->stats);
        struct RelGuard { rpq_result *r; ~RelGuard() { rpq_result_release(r); } } rg{rel};
        uint64_t nrel = rel->nrows;
        // (x, y) columns; backward results are (y, x) pairs sorted by (y, x)
        std::vector<uint32_t *> rc = backward ? std::vector<uint32_t *>{rel->cols[1], rel->cols[0]}
                                              : std::vector<uint32_t *>{rel->cols[0], rel->cols[1]};
        // own the columns in the pool (so compaction can replace them)
        for (auto &c : rc) {
            uint32_t *o2 = (uint32_t *)P.get(std::max<uint64_t>(nrel, 1) * 4);
            if (!o2) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            if (nrel) RPQ_CUDA_TRY(cudaMemcpyAsync(o2, c, nrel * 4, cudaMemcpyDeviceToDevice, s));
            c = o2;
        }
        // ---- filter by y's candidates (and s == d for x == y) ----
        if (nrel) {
            uint8_t *flag = (uint8_t *)P.get(nrel);
            if (!flag) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            k_pair_flags<<<grid_for(nrel), 256, 0, s>>>(rc[0], rc[1], nrel, pred(y), x == y ? 1 : 0, flag, pred(x),
                                                        backward ? 1 : 0);
            st = compact(P, rc, nrel, flag, s);
            if (st != RPQ_OK) return st;
        }
        // ---- join ----
        if (k == 0) {
            T.vars = {x};
            T.cols = {rc[0]};
            if (y != x) { T.vars.push_back(y); T.cols.push_back(rc[1]); }
            T.n = nrel;
            continue;
        }
        if (cx >= 0 && cy >= 0) {   // semi-join (relation sorted by (src,dst))
            if (T.n) {
                uint8_t *flag = (uint8_t *)P.get(T.n);
                if (!flag) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
                k_semijoin<<<grid_for(T.n), 256, 0, s>>>(T.cols[cx], T.cols[cy], T.n, rc[0], rc[1], nrel, flag);
                st = compact(P, T.cols, T.n, flag, s);
                if (st != RPQ_OK) return st;
            }
            continue;
        }
        // one endpoint bound: key column of the relation must be sorted
        const bool by_src = cx >= 0;
        uint32_t *rkey = rc[0], *rval = rc[1];
        if (!by_src && nrel && !backward) {       // (backward relations are already sorted by y)
            uint64_t *k1 = (uint64_t *)P.get(nrel * 8), *k2 = (uint64_t *)P.get(nrel * 8);
            if (!k1 || !k2) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            k_pack_swap<<<grid_for(nrel), 256, 0, s>>>(rc[0], rc[1], nrel, k1);
            size_t tb = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, tb, k1, k2, (int64_t)nrel, 0, 64, s);
            void *tmp = P.get(tb);
            if (!tmp) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            cub::DeviceRadixSort::SortKeys(tmp, tb, k1, k2, (int64_t)nrel, 0, 64, s);
            k_unpack<<<grid_for(nrel), 256, 0, s>>>(k2, nrel, rc[1], rc[0]);   // rc[1] = dst (key), rc[0] = src
            rkey = rc[1];
            rval = rc[0];
        } else if (!by_src) {
            rkey = rc[1];
            rval = rc[0];
        }
        const int ck = by_src ? cx : cy;
        const uint32_t newvar = by_src ? y : x;
        unsigned long long *lo = (unsigned long long *)P.get(std::max<uint64_t>(T.n, 1) * 8);
        unsigned long long *cnt = (unsigned long long *)P.get(std::max<uint64_t>(T.n, 1) * 8);
        unsigned long long *off = (unsigned long long *)P.get(std::max<uint64_t>(T.n, 1) * 8 + 8);
        if (!lo || !cnt || !off) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
        uint64_t total = 0;
        if (T.n) {
            k_join_count<<<grid_for(T.n), 256, 0, s>>>(T.cols[ck], T.n, rkey, nrel, lo, cnt);
            size_t tb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int64_t)T.n, s);
            void *tmp = P.get(tb);
            if (!tmp) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int64_t)T.n, s);
            unsigned long long a = 0, b = 0;
            RPQ_CUDA_TRY(cudaMemcpyAsync(&a, off + T.n - 1, 8, cudaMemcpyDeviceToHost, s));
            RPQ_CUDA_TRY(cudaMemcpyAsync(&b, cnt + T.n - 1, 8, cudaMemcpyDeviceToHost, s));
            RPQ_CUDA_TRY(cudaStreamSynchronize(s));
            total = a + b;
        }
        std::vector<uint32_t *> nc(T.cols.size() + 1);
        for (auto &c : nc) {
            c = (uint32_t *)P.get(std::max<uint64_t>(total, 1) * 4);
            if (!c) return rpq_fail(RPQ_ENOMEM, "crpq: out of device memory (%llu tuples)", (unsigned long long)total);
        }
        if (total) {
            uint32_t **d_in = (uint32_t **)P.get(T.cols.size() * sizeof(void *));
            uint32_t **d_out = (uint32_t **)P.get(nc.size() * sizeof(void *));
            if (!d_in || !d_out) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
            RPQ_CUDA_TRY(cudaMemcpyAsync(d_in, T.cols.data(), T.cols.size() * sizeof(void *), cudaMemcpyHostToDevice, s));
            RPQ_CUDA_TRY(cudaMemcpyAsync(d_out, nc.data(), nc.size() * sizeof(void *), cudaMemcpyHostToDevice, s));
            k_join_write<<<grid_for(T.n), 256, 0, s>>>(d_in, (uint32_t)T.cols.size(), T.n, lo, cnt, off, rval, d_out);
            RPQ_CUDA_TRY(cudaStreamSynchronize(s));
        }
        for (auto c : T.cols) P.put(c);
        T.cols = nc;
        T.vars.push_back(newvar);
        T.n = total;
    }

    // ---- distinct-vertex filters (CQ4/CQ5) ----
    if (q->num_distinct && T.n) {
        uint8_t *flag = (uint8_t *)P.get(T.n);
        if (!flag) return rpq_fail(RPQ_ENOMEM, "crpq: oom");
        RPQ_CUDA_TRY(cudaMemsetAsync(flag, 1, T.n, s));
        for (uint32_t i = 0; i < q->num_distinct; ++i) {
            const int a = T.col_of(q->distinct_pairs[2 * i]), b = T.col_of(q->distinct_pairs[2 * i + 1]);
            k_ne_flags<<<grid_for(T.n), 256, 0, s>>>(T.cols[a], T.cols[b], T.n, flag);
        }
        rpq_status st = compact(P, T.cols, T.n, flag, s);
        if (st != RPQ_OK) return st;
    }

    // ---- lexicographic order in output-variable order: stable LSD radix
    // passes; a projection (crpq_eval_project) then keeps distinct rows ----
    const uint32_t nout = (uint32_t)outv.size();
    const bool project = nout < nvars;
    rpq_result *res = new rpq_result();
    res->stream = (void *)s;
    res->alloc_snap = alloc_snapshot();
    res->device = g->device;
    res->ncols = nout;
    res->nrows = T.n;
    res->count = T.n;
    auto fail = [&](rpq_status st) { rpq_result_release(res); return st; };
    std::vector<uint32_t *> sorted(nout);
    for (uint32_t k = 0; k < nout; ++k) {
        sorted[k] = (uint32_t *)P.get(std::max<uint64_t>(T.n, 1) * 4);
        if (!sorted[k]) return fail(rpq_fail(RPQ_ENOMEM, "crpq: out of device memory (result)"));
    }
    if (T.n) {
        uint32_t *perm = (uint32_t *)P.get(T.n * 4), *perm2 = (uint32_t *)P.get(T.n * 4);
        uint32_t *key = (uint32_t *)P.get(T.n * 4), *key2 = (uint32_t *)P.get(T.n * 4);
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, perm, perm2, (int64_t)T.n, 0, 32, s);
        void *tmp = P.get(tb);
        if (!perm || !perm2 || !key || !key2 || !tmp) return fail(rpq_fail(RPQ_ENOMEM, "crpq: oom"));
        k_iota32<<<grid_for(T.n), 256, 0, s>>>(perm, T.n);
        for (int k = (int)nout - 1; k >= 0; --k) {
            const int c = T.col_of(outv[k]);
            k_gather<<<grid_for(T.n), 256, 0, s>>>(T.cols[c], perm, T.n, key);
            cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, perm, perm2, (int64_t)T.n, 0, 32, s);
            std::swap(perm, perm2);
        }
        for (uint32_t k = 0; k < nout; ++k)
            k_gather<<<grid_for(T.n), 256, 0, s>>>(T.cols[T.col_of(outv[k])], perm, T.n, sorted[k]);
    }
    uint64_t nres = T.n;
    if (project && nres) {
        uint8_t *flag = (uint8_t *)P.get(nres);
        uint32_t **d_c = (uint32_t **)P.get(nout * sizeof(void *));
        if (!flag || !d_c) return fail(rpq_fail(RPQ_ENOMEM, "crpq: oom"));
        RPQ_CUDA_TRY(cudaMemcpyAsync(d_c, sorted.data(), nout * sizeof(void *), cudaMemcpyHostToDevice, s));
        k_row_changed<<<grid_for(nres), 256, 0, s>>>(d_c, nout, nres, flag);
        rpq_status cs = compact(P, sorted, nres, flag, s);
        if (cs != RPQ_OK) return fail(cs);
    }
    res->nrows = res->count = nres;
    for (uint32_t k = 0; k < nout; ++k) {
        if (!dev_alloc_to(res->cols[k], std::max<uint64_t>(nres, 1) * 4, s)) {
            cudaGetLastError();
            return fail(rpq_fail(RPQ_ENOMEM, "crpq: out of device memory (result)"));
        }
        if (nres) RPQ_CUDA_TRY(cudaMemcpyAsync(res->cols[k], sorted[k], nres * 4, cudaMemcpyDeviceToDevice, s));
    }
    cudaEventRecord(e1, s);
    cudaError_t ce = cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ce != cudaSuccess) return fail(rpq_fail(RPQ_ECUDA, "crpq: %s", cudaGetErrorString(ce)));
    ST.total_ms = ms;
    ST.count = nres;
    res->stats = ST;
    *out = res;
    return RPQ_OK;
}

// Start-in-the-middle plan (WavePlan A3/A4): R(alpha m
// beta) for a middle label m, explored from the m-edges outwards -- alpha
// backwards (reversed automaton over in-edges, "with transpose") from the
// sources of m-edges, beta forwards from their targets -- then joined on the
// middle edge and projected to distinct (x, y).  The pairs cannot come out
// in source order during exploration ("result pairs cannot be confirmed in
// order of start vertices"), so they are enumerated, then sorted + deduped.
// Executed as the CRPQ x -alpha-> u, u -m-> w, w -beta-> y with the
// worst-case-optimal join (its matching order starts at u, w: the middle).
extern "C" rpq_status rpq_eval_middle(const rpq_graph *g, const char *alpha, const char *mid, const char *beta,
                                      const rpq_eval_opts *opts, rpq_result **out) {
    NvtxRange nvtx_("rpq_eval_middle");
    if (out) *out = nullptr;
    if (!g || !alpha || !mid || !beta || !out) return rpq_fail(RPQ_EINVAL, "rpq_eval_middle: NULL argument");
    rpq_nfa *na = nullptr, *nm = nullptr, *nb = nullptr;
    struct G3 { rpq_nfa **a, **b, **c; ~G3() { delete *a; delete *b; delete *c; } } gd{&na, &nm, &nb};
    size_t eo = 0;
    rpq_status st;
    if ((st = compile_regex(g->label_names, alpha, 0, &na, &eo)) != RPQ_OK) return st;
    if ((st = compile_regex(g->label_names, mid, 0, &nm, &eo)) != RPQ_OK) return st;
    if ((st = compile_regex(g->label_names, beta, 0, &nb, &eo)) != RPQ_OK) return st;
    const int32_t vl[4] = {-1, -1, -1, -1};
    const int64_t vc[4] = {-1, -1, -1, -1};
    const uint32_t ax[3] = {0, 1, 2}, ay[3] = {1, 2, 3};
    const rpq_nfa *an[3] = {na, nm, nb};
    crpq_query q{};
    q.num_vars = 4;
    q.var_label = vl;
    q.var_const = vc;
    q.num_atoms = 3;
    q.atom_x = ax;
    q.atom_y = ay;
    q.atom_nfa = an;
    rpq_eval_opts o{};
    if (opts) o = *opts;
    o.mode |= RPQ_WCOJ;
    const uint32_t ov[2] = {0, 3};
    return crpq_eval_project(g, &q, ov, 2, &o, out);
}
