// rpq_graph_load: host (src, dst, label) triples -> per-label device CSR.
//
// PAPER.md: G = (V, E, L) with labelled edges; LGF keeps "a
// separate grid ... for each edge label" so that traversal by edge label is
// direct.  Here that becomes one CSR per label (no grid,
// block or slice partitioning: the graphs fit in 180 GB of HBM).  E is a set
// of (u, l, w) triples (reading R4): duplicates are removed on the device.
//
// Build (one-time, excluded from query time as the paper excludes loading,
// P:1151): validate -> per-label counting scatter of 64-bit keys (u<<32|w)
// -> per-label radix sort (CUB) -> unique -> degree histogram + scan ->
// neighbour array.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "internal.h"

namespace {

__global__ void k_validate(const uint32_t *src, const uint32_t *dst, const uint16_t *lab, uint64_t ne,
                           uint32_t nv, uint32_t nl, int *bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne; i += (uint64_t)gridDim.x * blockDim.x)
        if (src[i] >= nv || dst[i] >= nv || (lab && lab[i] >= nl)) *bad = 1;
}

__global__ void k_label_hist(const uint16_t *lab, uint64_t ne, unsigned long long *cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t l = lab[i];
        // warp-aggregated increment: lanes with the same label elect a leader
        unsigned peers = __match_any_sync(__activemask(), l);
        int leader = __ffs(peers) - 1;
        if ((int)(threadIdx.x & 31) == leader) atomicAdd(&cnt[l], (unsigned long long)__popc(peers));
    }
}

__global__ void k_scatter(const uint32_t *src, const uint32_t *dst, const uint16_t *lab, uint64_t ne,
                          unsigned long long *cursor, uint64_t *keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t l = lab[i];
        unsigned peers = __match_any_sync(__activemask(), l);
        int leader = __ffs(peers) - 1;
        int lane = threadIdx.x & 31;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(&cursor[l], (unsigned long long)__popc(peers));
        base = __shfl_sync(peers, base, leader);
        uint64_t pos = base + __popc(peers & ((1u << lane) - 1));
        keys[pos] = ((uint64_t)src[i] << 32) | dst[i];
    }
}

// The unique-edge count m of the label stays on the device (no host round
// trip per label): the kernels read it.
__global__ void k_degree_nbr(const uint64_t *keys, const uint64_t *m_dev, uint32_t *deg, uint32_t *nbr,
                             uint32_t *mm, uint64_t *fl) {
    const uint64_t m = *m_dev;
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        const uint32_t w = (uint32_t)k;
        nbr[i] = w;
        atomicAdd(&deg[(k >> 32) + 1], 1u);
        lo = min(lo, w);
        hi = max(hi, w);
    }
    // destination range (reduced per warp, then one atomic per warp)
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) { atomicMin(mm, lo); atomicMax(mm + 1, hi); }
    if (blockIdx.x == 0 && threadIdx.x == 0 && m) { fl[0] = keys[0]; fl[1] = keys[m - 1]; }   // source range
}

// largest row of a label: max over v of off[v + 1] - off[v]
__global__ void k_max_deg(const uint32_t *off, uint32_t nv, uint32_t *out) {
    uint32_t m = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, off[v + 1] - off[v]);
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

inline int grid_for(uint64_t n, int block = 256) {
    uint64_t g = (n + block - 1) / block;
    if (g > 148ull * 32) g = 148ull * 32;
    if (g == 0) g = 1;
    return (int)g;
}

struct Cleanup {
    std::vector<void *> ptrs;
    cudaStream_t s;
    ~Cleanup() { for (void *p : ptrs) dev_free(p, s); }
};

}  // namespace

// Long-lived graph blocks: the caller's allocator when one was installed at
// load time (rpq_set_allocator), else plain cudaMalloc (not the stream pool:
// the graph outlives every stream the caller may use).
void *graph_alloc(const rpq_graph *g, size_t bytes, void *s) {
    if (g->alloc_snap && g->alloc_snap->alloc) return g->alloc_snap->alloc(bytes, (void *)s, g->alloc_snap->ctx);
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    return p;
}

void graph_block_free(const rpq_graph *g, void *p) {
    if (!p) return;
    if (g->alloc_snap && g->alloc_snap->free_) g->alloc_snap->free_(p, nullptr, g->alloc_snap->ctx);
    else cudaFree(p);
}

extern "C" void rpq_graph_free(rpq_graph *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    cudaDeviceSynchronize();         // no evaluation may still read the CSR
    for (int p = 0; p < 2; ++p) {    // label CSRs are slices of these blocks
        graph_block_free(g, g->off_base[p]);
        graph_block_free(g, g->nbr_base[p]);
    }
    graph_block_free(g, g->vlabel);
    graph_block_free(g, g->d_iota);
    for (void *b : g->extra_blocks) graph_block_free(g, b);
    for (auto *e : g->prod_cache) {
        graph_block_free(g, e->d_pidx);
        delete e;
    }
    delete g->alloc_snap;
    delete g;
    dev_available_invalidate();
}

extern "C" rpq_status rpq_graph_load(const rpq_graph_desc *d, rpq_graph **out) {
    NvtxRange nvtx_("rpq_graph_load");
    if (out) *out = nullptr;
    if (!d || !out) return rpq_fail(RPQ_EINVAL, "rpq_graph_load: NULL argument");
    if (d->num_vertices == 0) return rpq_fail(RPQ_EINVAL, "rpq_graph_load: num_vertices == 0");
    if (d->num_edges && (!d->src || !d->dst || !d->label))
        return rpq_fail(RPQ_EINVAL, "rpq_graph_load: NULL edge arrays");
    if (d->num_labels == 0 || d->num_labels > 65535 || !d->label_names)
        return rpq_fail(RPQ_EINVAL, "rpq_graph_load: bad label vocabulary");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return rpq_fail(RPQ_ECUDA, "rpq_graph_load: no CUDA device");
    }
    if (d->device < 0 || d->device >= ndev) return rpq_fail(RPQ_EINVAL, "rpq_graph_load: bad device");
    RPQ_CUDA_TRY(cudaSetDevice(d->device));
    cudaStream_t s = (cudaStream_t)d->cuda_stream;
    const uint64_t ne = d->num_edges;
    const uint32_t nv = d->num_vertices, nl = d->num_labels;

    Cleanup tmp{{}, s};
    auto alloc = [&](size_t bytes) { void *p = dev_alloc(bytes, s); if (p) tmp.ptrs.push_back(p); return p; };

    uint32_t *d_src = (uint32_t *)alloc(ne * 4), *d_dst = (uint32_t *)alloc(ne * 4);
    uint16_t *d_lab = (uint16_t *)alloc(ne * 2);
    int *d_bad = (int *)alloc(sizeof(int));
    unsigned long long *d_cnt = (unsigned long long *)alloc(nl * 8ull);
    uint64_t *keys = (uint64_t *)alloc(ne * 8), *keys2 = (uint64_t *)alloc(ne * 8);
    uint64_t *d_nsel = (uint64_t *)alloc(8);
    if (!d_src || !d_dst || !d_lab || !d_bad || !d_cnt || !keys || !keys2 || !d_nsel)
        return rpq_fail(RPQ_ENOMEM, "rpq_graph_load: out of device memory");
    if (ne) {
        RPQ_CUDA_TRY(cudaMemcpyAsync(d_src, d->src, ne * 4, cudaMemcpyHostToDevice, s));
        RPQ_CUDA_TRY(cudaMemcpyAsync(d_dst, d->dst, ne * 4, cudaMemcpyHostToDevice, s));
        RPQ_CUDA_TRY(cudaMemcpyAsync(d_lab, d->label, ne * 2, cudaMemcpyHostToDevice, s));
    }
    RPQ_CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
    RPQ_CUDA_TRY(cudaMemsetAsync(d_cnt, 0, nl * 8ull, s));
    if (ne) {
        k_validate<<<grid_for(ne), 256, 0, s>>>(d_src, d_dst, d_lab, ne, nv, nl, d_bad);
        k_label_hist<<<grid_for(ne), 256, 0, s>>>(d_lab, ne, d_cnt);
    }
    int bad = 0;
    std::vector<unsigned long long> cnt(nl);
    RPQ_CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    RPQ_CUDA_TRY(cudaMemcpyAsync(cnt.data(), d_cnt, nl * 8ull, cudaMemcpyDeviceToHost, s));
    RPQ_CUDA_TRY(cudaStreamSynchronize(s));
    if (bad) return rpq_fail(RPQ_EINVAL, "rpq_graph_load: vertex id >= num_vertices or label >= num_labels");
    // per-label offsets and CSR edge indices are u32 (internal.h LabelCSR)
    for (uint32_t l = 0; l < nl; ++l)
        if (cnt[l] > 0xffffffffull)
            return rpq_fail(RPQ_EUNSUPPORTED, "rpq_graph_load: label %u has %llu >= 2^32 edges (u32 CSR offsets)", l,
                            (unsigned long long)cnt[l]);
    std::vector<unsigned long long> start(nl + 1, 0);
    for (uint32_t l = 0; l < nl; ++l) start[l + 1] = start[l] + cnt[l];
    rpq_graph *g = new rpq_graph();
    g->alloc_snap = alloc_snapshot();
    g->device = d->device;
    g->nv = nv;
    for (uint32_t l = 0; l < nl; ++l) g->label_names.emplace_back(d->label_names[l] ? d->label_names[l] : "");
    g->csr.resize(nl);
    const bool in_edges = (d->flags & RPQ_GRAPH_IN_EDGES) != 0;
    if (in_edges) g->in_csr.resize(nl);
    int vbits = 1;
    while (vbits < 32 && (1ull << vbits) < nv) ++vbits;
    auto fail = [&](rpq_status st, const char *m) { rpq_graph_free(g); return rpq_fail(st, "rpq_graph_load: %s", m); };
    // CUDA errors after g exists free it (and its CSR blocks) before returning
#define GTRY(expr)                                                                               \
    do {                                                                                         \
        cudaError_t _e = (expr);                                                                 \
        if (_e != cudaSuccess) {                                                                 \
            char _m[512];                                                                        \
            snprintf(_m, sizeof(_m), "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
            return fail(_e == cudaErrorMemoryAllocation ? RPQ_ENOMEM : RPQ_ECUDA, _m);           \
        }                                                                                        \
    } while (0)

    // pass 0: out-edge CSR (keys u<<32|w); pass 1 (RPQ_GRAPH_IN_EDGES): the
    // in-edge CSR of the transposed graph (keys w<<32|u), same construction.
    // One allocation for all labels' offsets and one for all neighbour
    // arrays (label slices 16-byte aligned, sized by the pre-dedup counts);
    // per-label results stay on the device and are read back once per pass.
    std::vector<uint64_t> nstart(nl + 1, 0);
    for (uint32_t l = 0; l < nl; ++l) nstart[l + 1] = nstart[l] + ((cnt[l] + 3) / 4) * 4;
    uint64_t *d_m = (uint64_t *)alloc(nl * 8ull), *d_fl = (uint64_t *)alloc(nl * 16ull);
    uint32_t *d_mm = (uint32_t *)alloc(nl * 8ull), *d_md = (uint32_t *)alloc(nl * 4ull);
    if (!d_m || !d_fl || !d_mm || !d_md) return fail(RPQ_ENOMEM, "out of device memory");
    // CUB temporary storage: the largest need over the labels, allocated once
    size_t tbytes = 0;
    for (uint32_t l = 0; l < nl; ++l) {
        if (!cnt[l]) continue;
        size_t t1 = 0, t2 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, t1, keys, keys2, (int64_t)cnt[l], 0, 32 + vbits, s);
        cub::DeviceSelect::Unique(nullptr, t2, keys2, keys, d_m, (int64_t)cnt[l], s);
        tbytes = std::max(tbytes, std::max(t1, t2));
    }
    {
        size_t t3 = 0;
        cub::DeviceScan::InclusiveSum(nullptr, t3, (uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)nv + 1, s);
        tbytes = std::max(tbytes, t3);
    }
    void *tstore = alloc(std::max<size_t>(tbytes, 16));
    if (!tstore) return fail(RPQ_ENOMEM, "sort temp");
    for (int pass = 0; pass < (in_edges ? 2 : 1); ++pass) {
        GTRY(cudaMemcpyAsync(d_cnt, start.data(), nl * 8ull, cudaMemcpyHostToDevice, s));
        if (ne) {
            if (pass == 0) k_scatter<<<grid_for(ne), 256, 0, s>>>(d_src, d_dst, d_lab, ne, d_cnt, keys);
            else k_scatter<<<grid_for(ne), 256, 0, s>>>(d_dst, d_src, d_lab, ne, d_cnt, keys);
        }
        GTRY(cudaGetLastError());
        std::vector<LabelCSR> &csrs = pass == 0 ? g->csr : g->in_csr;
        uint32_t *&off_all = g->off_base[pass];
        uint32_t *&nbr_all = g->nbr_base[pass];
        off_all = (uint32_t *)graph_alloc(g, (uint64_t)nl * (nv + 1ull) * 4, s);
        nbr_all = (uint32_t *)graph_alloc(g, std::max<uint64_t>(nstart[nl], 4) * 4, s);
        if (!off_all || !nbr_all) return fail(RPQ_ENOMEM, "CSR arrays");
        GTRY(cudaMemsetAsync(off_all, 0, (uint64_t)nl * (nv + 1ull) * 4, s));
        GTRY(cudaMemsetAsync(d_m, 0, nl * 8ull, s));
        GTRY(cudaMemsetAsync(d_fl, 0, nl * 16ull, s));
        GTRY(cudaMemsetAsync(d_mm, 0xff, nl * 8ull, s));   // (min, max) = (~0, ~0): max fixed below
        GTRY(cudaMemsetAsync(d_md, 0, nl * 4ull, s));
        for (uint32_t l = 0; l < nl; ++l) {
            LabelCSR &c = csrs[l];
            c.off = off_all + (uint64_t)l * (nv + 1ull);
            c.nbr = nbr_all + nstart[l];
            const uint64_t n = cnt[l];
            if (n == 0) continue;
            uint64_t *kin = keys + start[l], *kout = keys2 + start[l];
            size_t tb = tbytes;
            GTRY(cudaMemsetAsync(d_mm + 2 * l + 1, 0, 4, s));
            cub::DeviceRadixSort::SortKeys(tstore, tb, kin, kout, (int64_t)n, 0, 32 + vbits, s);
            tb = tbytes;
            cub::DeviceSelect::Unique(tstore, tb, kout, kin, d_m + l, (int64_t)n, s);
            k_degree_nbr<<<grid_for(n), 256, 0, s>>>(kin, d_m + l, c.off, c.nbr, d_mm + 2 * l, d_fl + 2 * l);
            tb = tbytes;
            cub::DeviceScan::InclusiveSum(tstore, tb, c.off, c.off, (int64_t)nv + 1, s);
            k_max_deg<<<grid_for(nv), 256, 0, s>>>(c.off, nv, d_md + l);
        }
        std::vector<uint64_t> hm(nl), hfl(2 * nl);
        std::vector<uint32_t> hmm(2 * nl), hmd(nl);
        GTRY(cudaMemcpyAsync(hmd.data(), d_md, nl * 4ull, cudaMemcpyDeviceToHost, s));
        GTRY(cudaMemcpyAsync(hm.data(), d_m, nl * 8ull, cudaMemcpyDeviceToHost, s));
        GTRY(cudaMemcpyAsync(hfl.data(), d_fl, nl * 16ull, cudaMemcpyDeviceToHost, s));
        GTRY(cudaMemcpyAsync(hmm.data(), d_mm, nl * 8ull, cudaMemcpyDeviceToHost, s));
        GTRY(cudaStreamSynchronize(s));
        for (uint32_t l = 0; l < nl; ++l) {
            LabelCSR &c = csrs[l];
            c.m = cnt[l] ? hm[l] : 0;
            c.max_deg = c.m ? hmd[l] : 0;
            if (!c.m) continue;              // empty label: min > max (defaults)
            c.src_min = (uint32_t)(hfl[2 * l] >> 32);
            c.src_max = (uint32_t)(hfl[2 * l + 1] >> 32);
            c.dst_min = hmm[2 * l];
            c.dst_max = hmm[2 * l + 1];
            if (pass == 0) g->ne += c.m;
        }
    }
    if (d->vertex_label) {
        if (d->num_vertex_labels && d->vertex_label_names)
            for (uint32_t i = 0; i < d->num_vertex_labels; ++i)
                g->vlabel_names.emplace_back(d->vertex_label_names[i] ? d->vertex_label_names[i] : "");
        g->h_vlabel.assign(d->vertex_label, d->vertex_label + nv);
        g->vlabel = (uint16_t *)graph_alloc(g, nv * 2ull, s);
        if (!g->vlabel) return fail(RPQ_ENOMEM, "vertex labels");
        GTRY(cudaMemcpyAsync(g->vlabel, d->vertex_label, nv * 2ull, cudaMemcpyHostToDevice, s));
    }
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(RPQ_ECUDA, cudaGetErrorString(e));
    *out = g;
    dev_available_invalidate();
    return RPQ_OK;
#undef GTRY
}

__global__ void k_pack_pairs(const uint32_t *a, const uint32_t *b, uint64_t n, uint64_t *key) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        key[i] = ((uint64_t)a[i] << 32) | b[i];
}

// One derived label's CSR (and its transpose when the graph keeps in-edges)
// from device pairs: pack -> radix sort -> unique -> degrees -> scan, as in
// rpq_graph_load.
static rpq_status build_derived_csr(rpq_graph *g, const uint32_t *ds, const uint32_t *dd, uint64_t n, bool transpose,
                                    LabelCSR &c, cudaStream_t s) {
    const uint32_t nv = g->nv;
    Cleanup tmp{{}, s};
    auto alloc = [&](size_t bytes) { void *p = dev_alloc(bytes, s); if (p) tmp.ptrs.push_back(p); return p; };
    uint64_t *k1 = (uint64_t *)alloc(std::max<uint64_t>(n, 1) * 8), *k2 = (uint64_t *)alloc(std::max<uint64_t>(n, 1) * 8);
    uint64_t *d_m = (uint64_t *)alloc(8), *d_fl = (uint64_t *)alloc(16);
    uint32_t *d_mm = (uint32_t *)alloc(8), *d_md = (uint32_t *)alloc(4);
    if (!k1 || !k2 || !d_m || !d_fl || !d_mm || !d_md) return rpq_fail(RPQ_ENOMEM, "rpq_graph_add_label: out of device memory");
    uint32_t *off = (uint32_t *)graph_alloc(g, (nv + 1ull) * 4, s);
    uint32_t *nbr = (uint32_t *)graph_alloc(g, std::max<uint64_t>(n, 4) * 4, s);
    if (off) g->extra_blocks.push_back(off);
    if (nbr) g->extra_blocks.push_back(nbr);
    if (!off || !nbr) return rpq_fail(RPQ_ENOMEM, "rpq_graph_add_label: out of device memory (CSR)");
    int vbits = 1;
    while (vbits < 32 && (1ull << vbits) < nv) ++vbits;
    RPQ_CUDA_TRY(cudaMemsetAsync(off, 0, (nv + 1ull) * 4, s));
    RPQ_CUDA_TRY(cudaMemsetAsync(d_m, 0, 8, s));
    RPQ_CUDA_TRY(cudaMemsetAsync(d_fl, 0, 16, s));
    RPQ_CUDA_TRY(cudaMemsetAsync(d_mm, 0xff, 4, s));
    RPQ_CUDA_TRY(cudaMemsetAsync(d_mm + 1, 0, 4, s));
    RPQ_CUDA_TRY(cudaMemsetAsync(d_md, 0, 4, s));
    if (n) {
        if (transpose) k_pack_pairs<<<grid_for(n), 256, 0, s>>>(dd, ds, n, k1);
        else k_pack_pairs<<<grid_for(n), 256, 0, s>>>(ds, dd, n, k1);
        size_t t1 = 0, t2 = 0, t3 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, t1, k1, k2, (int64_t)n, 0, 32 + vbits, s);
        cub::DeviceSelect::Unique(nullptr, t2, k2, k1, d_m, (int64_t)n, s);
        cub::DeviceScan::InclusiveSum(nullptr, t3, off, off, (int64_t)nv + 1, s);
        void *ts = alloc(std::max(t1, std::max(t2, t3)));
        if (!ts) return rpq_fail(RPQ_ENOMEM, "rpq_graph_add_label: sort temp");
        size_t tb = t1;
        cub::DeviceRadixSort::SortKeys(ts, tb, k1, k2, (int64_t)n, 0, 32 + vbits, s);
        tb = t2;
        cub::DeviceSelect::Unique(ts, tb, k2, k1, d_m, (int64_t)n, s);
        k_degree_nbr<<<grid_for(n), 256, 0, s>>>(k1, d_m, off, nbr, d_mm, d_fl);
        tb = t3;
        cub::DeviceScan::InclusiveSum(ts, tb, off, off, (int64_t)nv + 1, s);
        k_max_deg<<<grid_for(nv), 256, 0, s>>>(off, nv, d_md);
    }
    uint64_t hm = 0, hfl[2] = {0, 0};
    uint32_t hmm[2] = {0, 0}, hmd = 0;
    RPQ_CUDA_TRY(cudaMemcpyAsync(&hm, d_m, 8, cudaMemcpyDeviceToHost, s));
    RPQ_CUDA_TRY(cudaMemcpyAsync(hfl, d_fl, 16, cudaMemcpyDeviceToHost, s));
    RPQ_CUDA_TRY(cudaMemcpyAsync(hmm, d_mm, 8, cudaMemcpyDeviceToHost, s));
    RPQ_CUDA_TRY(cudaMemcpyAsync(&hmd, d_md, 4, cudaMemcpyDeviceToHost, s));
    RPQ_CUDA_TRY(cudaStreamSynchronize(s));
    c = LabelCSR{};
    c.off = off;
    c.nbr = nbr;
    c.m = n ? hm : 0;
    c.max_deg = c.m ? hmd : 0;
    if (c.m) {
        c.src_min = (uint32_t)(hfl[0] >> 32);
        c.src_max = (uint32_t)(hfl[1] >> 32);
        c.dst_min = hmm[0];
        c.dst_max = hmm[1];
    }
    return RPQ_OK;
}

extern "C" rpq_status rpq_graph_add_label(rpq_graph *g, const char *name, const uint32_t *src, const uint32_t *dst,
                                          uint64_t n, int on_device, void *stream, uint32_t *label_id) {
    if (!g || !name || !*name || (n && (!src || !dst))) return rpq_fail(RPQ_EINVAL, "rpq_graph_add_label: bad argument");
    for (const auto &l : g->label_names)
        if (l == name) return rpq_fail(RPQ_EINVAL, "rpq_graph_add_label: label '%s' exists", name);
    if (g->label_names.size() >= 65535) return rpq_fail(RPQ_EUNSUPPORTED, "rpq_graph_add_label: too many labels");
    if (n > 0xffffffffull) return rpq_fail(RPQ_EUNSUPPORTED, "rpq_graph_add_label: >= 2^32 edges (u32 CSR offsets)");
    RPQ_CUDA_TRY(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)stream;
    Cleanup tmp{{}, s};
    const uint32_t *ds = src, *dd = dst;
    if (!on_device && n) {
        uint32_t *a = (uint32_t *)dev_alloc(n * 4, s), *b = (uint32_t *)dev_alloc(n * 4, s);
        if (a) tmp.ptrs.push_back(a);
        if (b) tmp.ptrs.push_back(b);
        if (!a || !b) return rpq_fail(RPQ_ENOMEM, "rpq_graph_add_label: out of device memory");
        RPQ_CUDA_TRY(cudaMemcpyAsync(a, src, n * 4, cudaMemcpyHostToDevice, s));
        RPQ_CUDA_TRY(cudaMemcpyAsync(b, dst, n * 4, cudaMemcpyHostToDevice, s));
        ds = a;
        dd = b;
    }
    int *d_bad = (int *)dev_alloc(sizeof(int), s);
    if (!d_bad) return rpq_fail(RPQ_ENOMEM, "rpq_graph_add_label: out of device memory");
    tmp.ptrs.push_back(d_bad);
    int bad = 0;
    RPQ_CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
    if (n) k_validate<<<grid_for(n), 256, 0, s>>>(ds, dd, nullptr, n, g->nv, 1, d_bad);
    RPQ_CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    RPQ_CUDA_TRY(cudaStreamSynchronize(s));
    if (bad) return rpq_fail(RPQ_EINVAL, "rpq_graph_add_label: vertex id >= num_vertices");
    LabelCSR out_c, in_c;
    rpq_status st = build_derived_csr(g, ds, dd, n, false, out_c, s);
    if (st != RPQ_OK) return st;
    const bool in_edges = g->in_csr.size() == g->csr.size() && !g->csr.empty();
    if (in_edges && (st = build_derived_csr(g, ds, dd, n, true, in_c, s)) != RPQ_OK) return st;
    {
        std::lock_guard<std::mutex> lk(g->sym_mu);
        g->csr.push_back(out_c);
        if (in_edges) g->in_csr.push_back(in_c);
        g->label_names.emplace_back(name);
        g->ne += out_c.m;
        if (!g->sym.empty()) g->sym.push_back(-1);
    }
    if (label_id) *label_id = (uint32_t)(g->label_names.size() - 1);
    dev_available_invalidate();
    return RPQ_OK;
}

extern "C" rpq_status rpq_graph_info(const rpq_graph *g, uint32_t *nv, uint64_t *ne, uint32_t *nl) {
    if (!g) return rpq_fail(RPQ_EINVAL, "NULL graph");
    if (nv) *nv = g->nv;
    if (ne) *ne = g->ne;
    if (nl) *nl = (uint32_t)g->csr.size();
    return RPQ_OK;
}

extern "C" rpq_status rpq_graph_label_csr(const rpq_graph *g, uint32_t l, const uint32_t **off,
                                          const uint32_t **nbr, uint64_t *m) {
    if (!g || l >= g->csr.size()) return rpq_fail(RPQ_EINVAL, "bad graph/label");
    if (off) *off = g->csr[l].off;
    if (nbr) *nbr = g->csr[l].nbr;
    if (m) *m = g->csr[l].m;
    return RPQ_OK;
}
