// RPQ evaluation on sm_100a: level-synchronous, bit-parallel multi-source
// BFS over the product graph G x A(rho).
//
// PAPER.md (P:n = line n of /root/reference/PAPER.md):
//   Definition 1: the result is the set of DISTINCT (x, y) such
//     that a path x -> ... -> y has a label word in L(rho).
//   Automata-based approach: traverse (vertex, state) pairs from
//     (x, q_init); a per-source visited set over (vertex, state) keeps the
//     output distinct and the traversal finite; a pair is emitted when a
//     final state is reached.
//   Challenge 2: the visited set costs |V||Q|/8 bytes per source;
//     the number of concurrent sources is bounded by memory.
//
// B200 design (DESIGN.md has the full rationale and the roofline):
//   * One bit per source.  A batch of B sources is a column block of
//     nw = ceil(B/64) 64-bit words.  Two state arrays, row-major
//     word[row * nw + w], one row per (state q, vertex v in range_q):
//     Vis (every reached bit) and Done (bits already expanded).  range_q is
//     the hull of the destination ranges of the labels entering q (plus the
//     batch's sources for q0; q0 gets no rows when nothing enters it).
//   * A level is one k_level launch inside a device-driven loop (a CUDA graph
//     with a conditional WHILE node).  A warp owns one active (row, 32-chunk
//     block): it advances up to 8 chunks at once (f = Vis & ~Done; Done |= f,
//     the row's single owner writes Done) and walks the row's per-label CSR
//     once for all of them, keeping 8 visited-word loads in flight per lane.
//   * Discovery: m = f & ~Vis[t]; Vis[t] |= m with red.or (no return value,
//     and the same sector the test just loaded, so it hits L2); the target's
//     chunk is marked in the next level's activity bitmaps (X per row word,
//     XB per 32 X words).  k_units lists the active units of each level for
//     dynamic fetching.  Bits OR-ed into a row before its owner reads Vis in
//     the same level are expanded early; each bit is still expanded once.
//   * Rows with more than HUB_EDGES neighbours for a transition are split
//     into HUB_EDGES segments processed by k_level_hub (degree skew).
//   * Touched (row, chunk) sets let sparse batches clear and count only what
//     they touched instead of dense memsets.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cmath>
#include <string>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <vector>

#include "internal.h"

namespace cg = cooperative_groups;

namespace {

constexpr int MAXQ = RPQ_MAX_STATES;
constexpr int MAXT = RPQ_MAX_TRANSITIONS;
constexpr int MAXL = RPQ_MAX_QUERY_LABELS;
constexpr uint32_t HUB_EDGES = 512;      // edges per hub segment
constexpr int TILE_V = 512;              // vertices per extraction tile
constexpr int NSTAT = 14;
#ifndef RPQ_LEVEL_MINB
#define RPQ_LEVEL_MINB 5
#endif
#ifndef RPQ_HUB_MINB
#define RPQ_HUB_MINB 4
#endif
#ifndef RPQ_LS_MAX
#define RPQ_LS_MAX 5          // a work unit splits into at most 2^RPQ_LS_MAX tickets ...
#endif
#ifndef RPQ_LS_WARPS
#define RPQ_LS_WARPS 8        // ... until there are RPQ_LS_WARPS tickets per warp of the grid
#endif
#ifndef RPQ_SLOTS
#define RPQ_SLOTS 8
#endif
constexpr int SLOTS = RPQ_SLOTS;          // visited-word loads in flight per lane
#ifndef RPQ_KGRP
#define RPQ_KGRP 8
#endif
constexpr int KGRP = RPQ_KGRP;          // chunks of a row advanced/expanded together (<= 8)

struct DevAuto {
    uint32_t nq;
    uint64_t final_mask;
    uint16_t toff[MAXQ + 1];
    uint8_t tslot[MAXT];
    uint8_t tto[MAXT];
    const uint32_t *off[MAXL];
    const uint32_t *nbr[MAXL];
    // pull (bottom-up) levels: transitions grouped by TARGET state and the
    // transposed CSR of every label slot (null when not loaded)
    uint16_t itoff[MAXQ + 1];
    uint8_t itfrom[MAXT];
    uint8_t itslot[MAXT];
    const uint32_t *ioff[MAXL];
    const uint32_t *inbr[MAXL];
};

struct Layout {
    uint64_t row_base[MAXQ];   // first row of state q
    uint32_t lo[MAXQ];         // range_q = [lo, lo + len)
    uint32_t len[MAXQ];
};

#ifndef RPQ_HUB_LOADS
#define RPQ_HUB_LOADS 512      // visited-word loads per lane in one hub record (edges x active chunks)
#endif
__host__ __device__ __forceinline__ uint32_t hub_seglen(int nk) {
    const uint32_t l = (uint32_t)RPQ_HUB_LOADS / (uint32_t)(nk > 0 ? nk : 1);
    return l < 32u ? 32u : (l > 512u ? 512u : l);      // <= HUB_EDGES
}

struct HubItem {                // a deferred row-group (frontier words in hubF)
    uint32_t row;              // global row (state, vertex)
    uint32_t xw;               // X word of the row (chunk block of 32)
    uint32_t nk;               // active chunks in the group (<= KGRP)
    uint64_t bits;             // chunk positions within the X word, 8 bits each
};

struct HubRec {                // one HUB_EDGES-edge segment of a long CSR row
    uint32_t hitem;
    uint32_t t;                // automaton transition
    uint32_t beg, end;         // CSR edge range
};

struct Ctrl {                  // per-level device counters / flags
    uint32_t active[2];        // "some row was activated" flag per level parity
    uint32_t nhub_items;
    uint32_t nhub_recs;
    uint32_t levels;           // levels run (device-side loop)
    uint32_t ucnt[2];          // active work units listed for the level of each parity
    uint32_t ucur[2];          // work-unit cursor (dynamic fetch) per parity
    uint32_t ntouched;         // entries of LevelArgs::TL
    uint32_t pcur[2];          // pull-level task cursor per parity
    uint32_t hcur;             // hub-record cursor (reset per level and before the seed hub launch)
    uint32_t blevel;           // levels of the current batch (reset by k_seed; the length bound)
    uint32_t txw;              // TX words that became non-zero in this batch (touched rows x 32 chunks)
};

// Clear / count a finished batch through its touched sets rather than
// densely?  Yes when few 32-X-word units were touched, or few X words (a
// row's 32-chunk block) even if most units were: R-MAT rows of vertices
// without in-edges under the query's labels are never touched, but they
// interleave with touched ones in every unit.
__device__ __forceinline__ bool sparse_batch(const Ctrl *c, uint64_t nunits, uint64_t nxwords) {
    return (uint64_t)c->ntouched * 4 <= nunits || (uint64_t)c->txw * 2 <= nxwords;
}

// One BFS level over the rows whose activity bit is set in (Xcur, XBcur).
//   row r = (state q, vertex v); word (r, col) holds 64 sources' bits.
//   X word (r, xw) = which 32-word chunks of the row are active;
//   XB bit (xi / 32) = some X word in [32 (xi/32), +32) is non-zero.
struct LevelArgs {
    uint64_t *Vis;             // visited: every reached bit, OR-ed in by red.or
    uint64_t *Done;            // bits already expanded (written only by the row's owner)
    // The fused advance is  f = Front & ~Mark;  Mark |= f  (row owner), and
    // discoveries are OR-ed into Disc.  Unbounded: Front = Disc = Vis,
    // Mark = Done.  Length-bounded (RPQ_BOUNDED, exact BFS levels, reading
    // D3): Front = N[par] (bits found by the previous level, zeroed when
    // consumed), Mark = Vis (written only by row owners), Disc = N[par ^ 1].
    uint64_t *Front, *Mark, *Disc;
    uint32_t bounded;
    uint32_t level_lim;        // last level of a batch (ctrl->blevel) that may expand; ~0u = unbounded
    uint32_t *Xcur, *Xnext;    // chunk-activity bitmaps, one word per (row, xw)
    uint32_t *XBcur, *XBnext;  // block bitmaps: one bit per 32 X words
    uint64_t nxwords;          // rows * nxw
    Ctrl *ctrl;
    int par;                   // level parity
    HubItem *hitems;
    uint64_t *hubF;            // [hitem][KGRP][32] frontier words
    HubRec *hrecs;
    uint32_t hitem_cap, hrec_cap;
    uint32_t nw;               // words per row
    uint32_t nxw;              // X words per row
    uint32_t cw;               // words per chunk (power of two <= 32)
    uint32_t *ulist;           // active work units of the level (k_units)
    uint32_t *TX;              // OR of all consumed X words of the batch (touched chunks)
    uint32_t *TU;              // touched work units of the batch (bitmap) ...
    uint32_t *TL;              // ... and their list (ctrl->ntouched entries)
    unsigned long long *stats;
    // direction-optimising levels: per column word, the sources
    // that may still gain bits (a superset: OR of the frontier words of the
    // level, or the exact new bits of a pull level); cur = this level's
    // filter, next = accumulated for the following level
    uint64_t *ActCur, *ActNext;
    uint64_t total_units;      // work units of the whole state (direction heuristic)
    uint32_t pull_mode;        // 0: top-down only; 1: bottom-up on dense levels
    uint32_t tma;              // 1: k_level<.., TMA = true> (bulk-copy expand ring)
};

// stats slots
enum { S_PE = 0, S_WORD_ITEMS, S_WORD_EDGE, S_ITEMS, S_ITEM_EDGES, S_ITEM_TRANS, S_X_RED, S_N_RED, S_PULL_LEVELS,
       S_PULL_LOADS, S_PULL_WORDS, S_PE_POST, S_ADV_WORDS, S_ADV_ZERO_SECTORS };

__device__ __forceinline__ uint64_t ld_cg(const uint64_t *p) { return __ldcg((const unsigned long long *)p); }

// fire-and-forget reductions (RED: no return value, the warp never waits)
__device__ __forceinline__ void red_or64(uint64_t *p, uint64_t v) {
    asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_or32(uint32_t *p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Direction of the level of parity p.par, decided identically by every kernel
// of the level from the active-unit count that k_units produced.
// Bottom-up when enabled for the query (symmetric relations, or forced) and
// at least 10 % of the work units are active (a dense frontier).
__device__ __forceinline__ bool level_pull(const LevelArgs &p) {
    if (!p.pull_mode) return false;
    const uint32_t n = *(volatile const uint32_t *)&p.ctrl->ucnt[p.par];
    return n != 0 && (uint64_t)n * 10ull > p.total_units;
}

// per-CTA accumulation of the activity columns in shared memory, flushed with
// one global OR per word and CTA (the column words are few and hot)
constexpr uint32_t ACT_SMEM_WORDS = 2048;
__device__ __forceinline__ void act_init(unsigned long long *actS, uint32_t nw) {
    for (uint32_t i = threadIdx.x; i < nw && i < ACT_SMEM_WORDS; i += blockDim.x) actS[i] = 0ull;
    __syncthreads();
}
__device__ __forceinline__ void act_or(unsigned long long *actS, uint64_t *g, uint32_t col, uint64_t m) {
    if (col < ACT_SMEM_WORDS) atomicOr(actS + col, (unsigned long long)m);
    else red_or64(g + col, m);
}
__device__ __forceinline__ void act_flush(const unsigned long long *actS, uint64_t *g, uint32_t nw) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nw && i < ACT_SMEM_WORDS; i += blockDim.x)
        if (actS[i]) red_or64(g + i, actS[i]);
}

// the per-batch layout lives in device memory (so a captured level graph is
// reusable across batches); each CTA stages it in shared memory
__device__ __forceinline__ void load_layout(Layout &S, const Layout *__restrict__ Sg, uint32_t nq) {
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
        S.row_base[q] = Sg->row_base[q];
        S.lo[q] = Sg->lo[q];
        S.len[q] = Sg->len[q];
    }
    __syncthreads();
}

__device__ __forceinline__ int row_state(const Layout &S, uint32_t nq, uint64_t row) {
    int q = 0;
    while (q + 1 < (int)nq && S.row_base[q + 1] <= row) ++q;
    return q;
}

// Before every level: list the active work units (set bits of XBcur, one
// unit = 32 X words) for dynamic fetching, clear XBcur, and reset the
// counters of the other parity / the hub buffers.  Block 0 does the resets.
__global__ void k_units(const LevelArgs p, uint64_t nxbwords) {
    const int par = p.par;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.ctrl->ucnt[par ^ 1] = 0;
        p.ctrl->ucur[par ^ 1] = 0;
        p.ctrl->pcur[par] = 0;
        p.ctrl->active[par ^ 1] = 0;   // set by this level's activations

        p.ctrl->nhub_items = 0;
        p.ctrl->nhub_recs = 0;
        p.ctrl->hcur = 0;
        p.ctrl->levels += 1;
        p.ctrl->blevel += 1;
    }
    if (p.pull_mode)   // the previous level's filter, free now: this level accumulates into it
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.nw; i += (uint64_t)gridDim.x * blockDim.x)
            p.ActNext[i] = 0ull;
    const int lane = threadIdx.x & 31;
    for (uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull; w0 < nxbwords;
         w0 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = w0 + lane;
        uint32_t x = w < nxbwords ? __ldcg(p.XBcur + w) : 0u;
        if (x) p.XBcur[w] = 0u;
        // units seen for the first time in this batch -> touched list (the
        // TU word w holds exactly the units of XB word w: one owner here)
        uint32_t fresh = 0;
        if (x) {
            const uint32_t tu = p.TU[w];
            fresh = x & ~tu;
            if (fresh) p.TU[w] = tu | fresh;
        }
        const int c = __popc(x);
        const int cf = __popc(fresh);
        int incl = c, inclf = cf;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            const int yf = __shfl_up_sync(0xffffffffu, inclf, o);
            if (lane >= o) { incl += y; inclf += yf; }
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        const int totf = __shfl_sync(0xffffffffu, inclf, 31);
        if (!tot) continue;
        uint32_t base = 0, basef = 0;
        if (lane == 31) {
            base = atomicAdd(&p.ctrl->ucnt[par], (uint32_t)tot);
            if (totf) basef = atomicAdd(&p.ctrl->ntouched, (uint32_t)totf);
        }
        base = __shfl_sync(0xffffffffu, base, 31) + (uint32_t)(incl - c);
        basef = __shfl_sync(0xffffffffu, basef, 31) + (uint32_t)(inclf - cf);
        while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            p.ulist[base++] = (uint32_t)(w * 32 + b);
        }
        while (fresh) {
            const int b = __ffs(fresh) - 1;
            fresh &= fresh - 1;
            p.TL[basef++] = (uint32_t)(w * 32 + b);
        }
    }
}

// ---- touched-set maintenance (sparse batches) ------------------------------
// A warp per touched unit (32 X words): zero the visited words of every
// chunk the batch touched, and the touched bitmaps, so the next batch starts
// clean without a dense memset of the whole state.
__global__ void k_clear_touched(const LevelArgs p, uint64_t nunits, int force_dense) {
    const uint32_t ntl = p.ctrl->ntouched;
    if (force_dense || !sparse_batch(p.ctrl, nunits, p.nxwords)) return;      // dense: k_clear_dense does it
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    for (uint64_t t = wid; t < ntl; t += nwarps) {
        const uint64_t u = p.TL[t];
        const uint64_t xi_l = u * 32 + lane;
        const uint32_t tx = xi_l < p.nxwords ? p.TX[xi_l] : 0u;
        if (tx) p.TX[xi_l] = 0u;
        if (lane == 0) p.TU[u >> 5] = 0u;
        unsigned todo = __ballot_sync(0xffffffffu, tx != 0);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            uint32_t x = __shfl_sync(0xffffffffu, tx, src);
            const uint64_t xi = u * 32 + src;
            const uint64_t row = xi / p.nxw;
            const uint32_t xw = (uint32_t)(xi % p.nxw);
            while (x) {
                const uint32_t bt = (uint32_t)(__ffs(x) - 1);
                x &= x - 1;
                const uint64_t col = (uint64_t)(xw * 32u + bt) * p.cw + lane;
                if (lane < (int)p.cw && col < p.nw) {
                    p.Vis[row * p.nw + col] = 0ull;
                    p.Done[row * p.nw + col] = 0ull;
                }
            }
        }
    }
}

// COUNT over the touched chunks only: bits of Vis[q][v][w] for final q that
// are not already set in a lower-numbered final state's row of v (the OR over
// final states, counted once).
// pe != nullptr: also the product edges of the touched chunks (popcount x
// product out-degree of (v, q), reading R12) -- every reached bit of a row
// with outgoing transitions lies in a touched chunk.
__device__ __forceinline__ uint32_t prod_deg(const DevAuto &A, int q, uint32_t v) {
    uint32_t d = 0;
    for (int t = A.toff[q]; t < A.toff[q + 1]; ++t) d += __ldg(A.off[A.tslot[t]] + v + 1) - __ldg(A.off[A.tslot[t]] + v);
    return d;
}

__global__ void __launch_bounds__(256, 3) k_count_touched(const DevAuto A, const Layout S, const LevelArgs p, uint64_t nunits,
                                unsigned long long *total, int force_dense, unsigned long long *pe = nullptr) {
    const uint32_t ntl = p.ctrl->ntouched;
    if (force_dense || !sparse_batch(p.ctrl, nunits, p.nxwords)) return;      // dense batch: k_count_total counts
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    unsigned long long acc = 0, pacc = 0;
    for (uint64_t t = wid; t < ntl; t += nwarps) {
        const uint64_t u = p.TL[t];
        const uint64_t xi_l = u * 32 + lane;
        const uint32_t tx = xi_l < p.nxwords ? p.TX[xi_l] : 0u;
        unsigned todo = __ballot_sync(0xffffffffu, tx != 0);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            uint32_t x = __shfl_sync(0xffffffffu, tx, src);
            const uint64_t xi = u * 32 + src;
            const uint64_t row = xi / p.nxw;
            const uint32_t xw = (uint32_t)(xi % p.nxw);
            const int q = row_state(S, A.nq, row);
            const bool fin = (A.final_mask >> q) & 1ull;
            const uint32_t v = S.lo[q] + (uint32_t)(row - S.row_base[q]);
            const uint32_t deg = pe ? prod_deg(A, q, v) : 0u;
            if (!fin && !deg) continue;
            // the row's touched chunks, 8 at a time with all their loads in
            // flight together (one chunk per round trip ran at 1.9 TB/s)
            while (x) {
                uint64_t w[8], lw[8];
                uint32_t col[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool has = x != 0;
                    const uint32_t bt = has ? (uint32_t)(__ffs(x) - 1) : 0u;
                    if (has) x &= x - 1;
                    col[k] = (xw * 32u + bt) * p.cw + (uint32_t)lane;
                    const bool ok = has && lane < (int)p.cw && col[k] < p.nw;
                    if (!ok) col[k] = 0xffffffffu;
                    w[k] = ok ? ld_cg(p.Vis + row * p.nw + col[k]) : 0ull;
                    lw[k] = 0ull;
                }
                // bits already counted in a lower-numbered final state's row
                // of v: loaded together with the row's own words (one round
                // trip, not two: the count pass ran at 3.8 TB/s on RMAT)
                if (fin)
                    for (int f = 0; f < q; ++f)
                        if (((A.final_mask >> f) & 1ull) && v - S.lo[f] < S.len[f]) {
                            const uint64_t fb = (S.row_base[f] + (v - S.lo[f])) * p.nw;
#pragma unroll
                            for (int k = 0; k < 8; ++k)
                                if (col[k] != 0xffffffffu) lw[k] |= ld_cg(p.Vis + fb + col[k]);
                        }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    pacc += (unsigned long long)__popcll(w[k]) * deg;
                    if (fin) acc += __popcll(w[k] & ~lw[k]);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        pacc += __shfl_xor_sync(0xffffffffu, pacc, o);
    }
    if (lane == 0 && acc) atomicAdd(total, acc);
    if (lane == 0 && pacc) atomicAdd(pe, pacc);
}

__global__ void k_level_end(Ctrl *ctrl, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, ctrl->active[0] ? 1u : 0u);   // activations of the parity-1 level
}


// Expand the edges [beg, end) of one CSR row for a group of up to KGRP
// active chunks of X word xw (chunk positions packed 8 bits each in `bits`).
// KC chunks x (8 / KC) edges are in flight per step, so every lane keeps 8
// independent visited-word loads outstanding.
//   m = f & ~Vis[t];  Vis[t] |= m (red, same sector as the test load, so it
//   hits L2);  X/XB activity of t (red).
template <int KC, bool STATS, bool BND = false>
__device__ __forceinline__ void expand_edges(const LevelArgs &p, const Layout &S, uint32_t q2,
                                             const uint32_t *__restrict__ nbr, uint32_t beg, uint32_t end,
                                             const uint64_t (&f)[KGRP], uint64_t bits, uint32_t xw, int lane,
                                             unsigned long long *st, bool &act, bool live) {
    constexpr int E = SLOTS / KC;
    const uint32_t tbase = (uint32_t)(S.row_base[q2] - S.lo[q2]);
    const uint32_t colbase = xw * 32u * p.cw + lane;
    int fpop = 0, nzw = 0;
#pragma unroll
    for (int k = 0; k < KC; ++k) { fpop += __popcll(f[k]); nzw += f[k] != 0; }
    uint32_t ckk[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) ckk[k] = ((uint32_t)(bits >> (8 * k)) & 0xffu) * p.cw;
    for (uint32_t j = beg; j < end; j += 32) {
        const uint32_t my = (j + lane < end) ? __ldg(nbr + j + lane) : 0u;
        const int cnt = (int)((end - j) < 32u ? (end - j) : 32u);
        // one step: issue all loads of E edges x KC chunks, then the ORs
        struct Buf {
            uint32_t trow[E];
            uint64_t vis[E][KC];
        };
        auto issue = [&](Buf &b, int e0) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const bool ok = e0 + e < cnt;
                b.trow[e] = tbase + __shfl_sync(0xffffffffu, my, (e0 + e) & 31);
                const uint64_t rb = (uint64_t)b.trow[e] * p.nw + colbase;
#pragma unroll
                for (int k = 0; k < KC; ++k) b.vis[e][k] = (ok && f[k]) ? ld_cg(p.Vis + rb + ckk[k]) : ~0ull;
            }
        };
        auto process = [&](const Buf &b, int e0) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                uint32_t lm = 0;   // chunks of this lane with new bits
                const uint64_t rb = (uint64_t)b.trow[e] * p.nw + colbase;
#pragma unroll
                for (int k = 0; k < KC; ++k) {
                    const uint64_t m = (e0 + e < cnt) ? (f[k] & ~b.vis[e][k]) : 0ull;
                    if (m) {
                        red_or64((BND ? p.Disc : p.Vis) + rb + ckk[k], m);
                        lm |= 1u << ((bits >> (8 * k)) & 0xffu);
                        if (STATS) st[S_N_RED]++;
                    }
                }
                // one warp OR (REDUX) instead of a ballot per chunk
                const uint32_t newmask = live ? __reduce_or_sync(0xffffffffu, lm) : 0u;
                // a target state without outgoing transitions is never
                // expanded: its rows only collect result bits, no activity
                if (lane == 0 && newmask) {
                    // activity of the target row: fire-and-forget ORs (the
                    // words are idempotent; no test load on the critical path)
                    const uint64_t xi = (uint64_t)b.trow[e] * p.nxw + xw;
                    red_or32(p.Xnext + xi, newmask);
                    red_or32(p.XBnext + (xi >> 10), 1u << ((xi >> 5) & 31));
                    act = true;
                    if (STATS) st[S_X_RED]++;
                }
            }
        };
        // (double-buffering the steps was measured slower: more registers,
        // no gain -- the loop is not bound by the latency of one step)
        for (int e0 = 0; e0 < cnt; e0 += E) {
            Buf b;
            issue(b, e0);
            process(b, e0);
        }
        if (STATS && nzw) {
            st[S_WORD_EDGE] += (unsigned long long)nzw * cnt;
            st[S_PE] += (unsigned long long)fpop * cnt;
        }
        if (STATS && lane == 0) st[S_ITEM_EDGES] += cnt;
    }
}

template <bool STATS>
__device__ __forceinline__ void flush_stats(unsigned long long *st, unsigned long long *out) {
    if constexpr (STATS) {
#pragma unroll
        for (int i = 0; i < NSTAT; ++i) {
            unsigned long long x = st[i];
#pragma unroll
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) == 0 && x) atomicAdd(out + i, x);
        }
    }
}

// ---- TMA bulk-copy expand (sm_100a): the target-row segments of a row's
// edges are fetched by cp.async.bulk into a per-warp shared-memory ring
// (TMA_NS slots of up to KGRP chunks x 256 B), completion on an mbarrier per
// slot.  With KC = 8 active chunks the register path holds one edge's 8 words
// per lane in flight (a row with d edges costs d DRAM round trips); the ring
// keeps TMA_NS edges in flight without registers.
#ifndef RPQ_TMA_NS
#define RPQ_TMA_NS 4
#endif
constexpr int TMA_NS = RPQ_TMA_NS;
#ifndef RPQ_TMA_MINB
#define RPQ_TMA_MINB 3
#endif
constexpr uint32_t TMA_SLOT = KGRP * 32 * 8;          // bytes per slot (8 chunks of 32 words)
constexpr int TMA_WARPS = 8;
constexpr uint32_t TMA_WARP_BYTES = TMA_NS * TMA_SLOT + 64;
constexpr uint32_t TMA_SMEM = TMA_WARPS * TMA_WARP_BYTES;

__device__ __forceinline__ uint32_t smem_u32(const void *ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

struct TmaRing {
    uint64_t *buf;     // TMA_NS slots of TMA_SLOT bytes
    uint64_t *bar;     // TMA_NS mbarriers
    uint32_t phase;    // bit s = parity to wait for on slot s
};

// Same contract as expand_edges for a group whose nk active chunks lie in a
// window of <= KGRP chunks starting at chunk c0 (bits relative to the X word).
// The ring runs over the whole edge range [beg, end) (hub segments: up to 512
// edges), with the neighbour ids of the current and the next 32-edge window
// held in registers, so it never drains at window boundaries.
template <bool STATS>
__device__ __forceinline__ void expand_edges_tma(const LevelArgs &p, const Layout &S, uint32_t q2,
                                                 const uint32_t *__restrict__ nbr, uint32_t beg, uint32_t end,
                                                 const uint64_t (&f)[KGRP], uint64_t bits, int nk, uint32_t c0,
                                                 uint32_t span, uint32_t xw, int lane, unsigned long long *st,
                                                 bool &act, bool live, TmaRing &R) {
    const uint32_t tbase = (uint32_t)(S.row_base[q2] - S.lo[q2]);
    const uint32_t colw = (xw * 32u + c0) * 32u;            // first word of the window (cw == 32)
    const uint32_t bytes = span * 256u;
    if (beg >= end) return;
    uint32_t wbase = beg;
    uint32_t my_cur = (beg + lane < end) ? __ldg(nbr + beg + lane) : 0u;
    uint32_t my_nxt = (beg + 32 + lane < end) ? __ldg(nbr + beg + 32 + lane) : 0u;
    uint32_t trows[TMA_NS];
    auto issue = [&](uint32_t e) {   // edge e (absolute), e - wbase < 64
        const uint32_t d = e - wbase;
        const uint32_t a = __shfl_sync(0xffffffffu, my_cur, d & 31);
        const uint32_t b2 = __shfl_sync(0xffffffffu, my_nxt, d & 31);
        const uint32_t trow = tbase + (d < 32 ? a : b2);
        const int sl = (int)((e - beg) % TMA_NS);
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(R.bar + sl, bytes);
            bulk_g2s(R.buf + (size_t)sl * (TMA_SLOT / 8), p.Vis + (uint64_t)trow * p.nw + colw, bytes, R.bar + sl);
        }
#pragma unroll
        for (int s2 = 0; s2 < TMA_NS; ++s2)
            if (s2 == sl) trows[s2] = trow;
    };
    for (uint32_t e = beg; e < end && e < beg + TMA_NS; ++e) issue(e);
    for (uint32_t e = beg; e < end; ++e) {
        if (e == wbase + 32) {               // next window of neighbour ids
            wbase += 32;
            my_cur = my_nxt;
            my_nxt = (wbase + 32 + lane < end) ? __ldg(nbr + wbase + 32 + lane) : 0u;
        }
        const int sl = (int)((e - beg) % TMA_NS);
        while (!mbar_try(R.bar + sl, (R.phase >> sl) & 1u)) {
        }
        R.phase ^= 1u << sl;
        uint32_t trow = 0;
#pragma unroll
        for (int s2 = 0; s2 < TMA_NS; ++s2)
            if (s2 == sl) trow = trows[s2];
        const uint64_t *sb = R.buf + (size_t)sl * (TMA_SLOT / 8);
        const uint64_t rb = (uint64_t)trow * p.nw + colw + lane;
        uint32_t lm = 0;
        int nzw = 0, fpop = 0;
#pragma unroll
        for (int k = 0; k < KGRP; ++k) {
            if (k >= nk) break;
            const uint32_t ck = ((uint32_t)(bits >> (8 * k)) & 0xffu) - c0;
            const uint64_t m = f[k] & ~sb[ck * 32u + lane];
            if (m) {
                red_or64(p.Vis + rb + ck * 32u, m);
                lm |= 1u << (ck + c0);
                if (STATS) st[S_N_RED]++;
            }
            if (STATS) { nzw += f[k] != 0; fpop += __popcll(f[k]); }
        }
        if (STATS) { st[S_WORD_EDGE] += nzw; st[S_PE] += fpop; }
        const uint32_t newmask = live ? __reduce_or_sync(0xffffffffu, lm) : 0u;
        if (lane == 0 && newmask) {
            const uint64_t xi = (uint64_t)trow * p.nxw + xw;
            red_or32(p.Xnext + xi, newmask);
            red_or32(p.XBnext + (xi >> 10), 1u << ((xi >> 5) & 31));
            act = true;
            if (STATS) st[S_X_RED]++;
        }
        __syncwarp();                          // every lane has read the slot
        if (e + TMA_NS < end) issue(e + TMA_NS);
    }
    if (STATS && lane == 0) st[S_ITEM_EDGES] += end - beg;
}

template <bool STATS, bool BND = false>
__device__ __forceinline__ void dispatch_edges(int nk, const LevelArgs &p, const Layout &S, uint32_t q2,
                                               const uint32_t *nbr, uint32_t beg, uint32_t end,
                                               const uint64_t (&f)[KGRP], uint64_t bits, uint32_t xw, int lane,
                                               unsigned long long *st, bool &act, bool live) {
    if constexpr (KGRP > 4) {
        if (nk > 4) {
            expand_edges<8, STATS, BND>(p, S, q2, nbr, beg, end, f, bits, xw, lane, st, act, live);
            return;
        }
    }
    if (nk > 2) expand_edges<4, STATS, BND>(p, S, q2, nbr, beg, end, f, bits, xw, lane, st, act, live);
    else if (nk > 1) expand_edges<2, STATS, BND>(p, S, q2, nbr, beg, end, f, bits, xw, lane, st, act, live);
    else expand_edges<1, STATS, BND>(p, S, q2, nbr, beg, end, f, bits, xw, lane, st, act, live);
}

// Main level kernel: a warp owns one active X word = one row and up to 32 of
// its chunks; groups of KGRP active chunks are advanced (N -> Vis, fused:
// f = Vis & ~Done; Done |= f) and then expanded along every automaton
// transition of the row's state.  Work units (32 X words = one XB bit) are
// interleaved over warps.
template <bool STATS, bool BND = false, bool TMA = false>
__global__ void __launch_bounds__(256, TMA ? RPQ_TMA_MINB : RPQ_LEVEL_MINB) k_level(const DevAuto A, const Layout *__restrict__ Sg,
                                                                         const LevelArgs p) {
    if (level_pull(p)) return;                 // bottom-up level: k_pull_prep + k_pull
    if (BND && *(volatile const uint32_t *)&p.ctrl->blevel > p.level_lim) return;   // length bound reached
    __shared__ Layout S;
    __shared__ unsigned long long actS[TMA ? 1 : ACT_SMEM_WORDS];
    extern __shared__ __align__(128) unsigned char tma_dyn[];
    load_layout(S, Sg, A.nq);
    if (!TMA && p.pull_mode) act_init(actS, p.nw);
    const int lane = threadIdx.x & 31;
    TmaRing ring{};
    if constexpr (TMA) {
        unsigned char *wb = tma_dyn + (threadIdx.x >> 5) * TMA_WARP_BYTES;
        ring.bar = reinterpret_cast<uint64_t *>(wb);
        ring.buf = reinterpret_cast<uint64_t *>(wb + 64);
        if (lane == 0) {
            for (int sl = 0; sl < TMA_NS; ++sl) mbar_init(ring.bar + sl, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    const uint32_t nunits = *(volatile uint32_t *)&p.ctrl->ucnt[p.par];
    unsigned long long st[NSTAT] = {};
    bool act = false;
    (void)wid;
    // Few active units (small row counts, e.g. knows+ over 65 K persons, or
    // the narrow first/last levels): split each unit into 2^ls tickets of
    // 32 >> ls X words so that every warp of the grid gets work; a ticket is
    // one atomic on the level's cursor.
    int ls = 0;
    while (ls < RPQ_LS_MAX && ((uint64_t)nunits << ls) < nwarps * RPQ_LS_WARPS) ++ls;
    const uint32_t ntk = nunits << ls;
    const int part_lanes = 32 >> ls;
    for (;;) {
        uint32_t tk = 0;
        if (lane == 0) tk = atomicAdd(&p.ctrl->ucur[p.par], 1u);
        tk = __shfl_sync(0xffffffffu, tk, 0);
        if (tk >= ntk) break;
        const uint64_t u = p.ulist[tk >> ls];
        const bool mine = (lane / part_lanes) == (int)(tk & ((1u << ls) - 1u));
        const uint64_t xi_l = u * 32 + lane;
        const uint32_t xl = (mine && xi_l < p.nxwords) ? __ldcg(p.Xcur + xi_l) : 0u;
        bool fresh = false;
        if (xl) {
            p.Xcur[xi_l] = 0u;
            const uint32_t t0 = p.TX[xi_l];
            p.TX[xi_l] = t0 | xl;      // single owner per level; levels are ordered
            fresh = t0 == 0u;
        }
        {
            const unsigned fm = __ballot_sync(0xffffffffu, fresh);
            if (fm && lane == 0) atomicAdd(&p.ctrl->txw, (uint32_t)__popc(fm));
        }
        unsigned todo = __ballot_sync(0xffffffffu, xl != 0);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            uint32_t x = __shfl_sync(0xffffffffu, xl, src);
            const uint64_t xi = u * 32 + src;
            const uint64_t row = xi / p.nxw;
            const uint32_t xw = (uint32_t)(xi % p.nxw);
            const int q = row_state(S, A.nq, row);
            const uint32_t v = S.lo[q] + (uint32_t)(row - S.row_base[q]);
            const uint64_t rb = row * p.nw + xw * 32u * p.cw + lane;
            const bool lane_ok = lane < (int)p.cw;
            // prefetch the CSR row bounds of every transition of q (lane t
            // holds transition toff[q] + t) while the advance runs
            const int t0 = A.toff[q], ntr = A.toff[q + 1] - t0;
            uint32_t obeg = 0, oend = 0;
            if (lane < ntr) {
                const uint32_t *off = A.off[A.tslot[t0 + lane]];
                obeg = __ldg(off + v);
                oend = __ldg(off + v + 1);
            }
            while (x) {
                // take up to KGRP active chunks and advance them (fused):
                // f = Vis & ~Done (bits reached but not yet expanded),
                // Done |= f; all loads of the group are issued together
                uint64_t f[KGRP], dd[KGRP];
                uint64_t bits = 0;
                int nk = 0;
#pragma unroll
                for (int k = 0; k < KGRP; ++k) {
                    const bool has = x != 0;
                    const uint32_t bt = has ? (uint32_t)(__ffs(x) - 1) : 0u;
                    if (has) x &= x - 1;
                    nk += has;
                    bits |= (uint64_t)bt << (8 * k);
                    const bool ok = has && lane_ok && xw * 32u * p.cw + bt * p.cw + lane < p.nw;
                    f[k] = ok ? ld_cg((BND ? p.Front : p.Vis) + rb + bt * p.cw) : 0ull;
                    dd[k] = ok ? (BND ? p.Mark : p.Done)[rb + bt * p.cw] : ~0ull;
                }
#pragma unroll
                for (int k = 0; k < KGRP; ++k) {
                    const uint32_t bt = (uint32_t)(bits >> (8 * k)) & 0xffu;
                    if (BND && f[k]) p.Front[rb + bt * p.cw] = 0ull;   // N[par] consumed
                    f[k] &= ~dd[k];
                    if (f[k]) {
                        (BND ? p.Mark : p.Done)[rb + bt * p.cw] = dd[k] | f[k];
                        // sources of this frontier word may gain bits next level
                        if (!TMA && p.pull_mode) act_or(actS, p.ActNext, (uint32_t)(rb - row * p.nw) + bt * p.cw, f[k]);
                        if (STATS) st[S_WORD_ITEMS]++;
                    }
                }
                if constexpr (STATS) {   // advance reads vs 32-byte sectors without frontier bits
#pragma unroll
                    for (int k = 0; k < KGRP; ++k) {
                        const uint32_t bt = (uint32_t)(bits >> (8 * k)) & 0xffu;
                        const bool okk = k < nk && lane_ok && xw * 32u * p.cw + bt * p.cw + lane < p.nw;
                        const unsigned vm = __ballot_sync(0xffffffffu, okk);
                        const unsigned nzm = __ballot_sync(0xffffffffu, okk && f[k] != 0);
                        if (lane == 0) {
                            st[S_ADV_WORDS] += __popc(vm);
                            for (int sct = 0; sct < 8; ++sct)
                                if (((vm >> (4 * sct)) & 15u) && !((nzm >> (4 * sct)) & 15u)) st[S_ADV_ZERO_SECTORS]++;
                        }
                    }
                }
                bool anyk = false;
#pragma unroll
                for (int k = 0; k < KGRP; ++k) anyk |= f[k] != 0;
                if (!__ballot_sync(0xffffffffu, anyk)) continue;
                if (STATS && lane == 0) st[S_ITEMS]++;
                int hslot = -1;
                for (int t = t0; t < t0 + ntr; ++t) {
                    const int slot = A.tslot[t];
                    uint32_t beg, end;
                    if (t - t0 < 32) {
                        beg = __shfl_sync(0xffffffffu, obeg, t - t0);
                        end = __shfl_sync(0xffffffffu, oend, t - t0);
                    } else {
                        beg = __ldg(A.off[slot] + v);
                        end = __ldg(A.off[slot] + v + 1);
                    }
                    if (STATS && lane == 0) st[S_ITEM_TRANS]++;
                    if (end == beg) continue;
                    if (end - beg > HUB_EDGES) {
                        if (hslot < 0) {
                            uint32_t hs = 0;
                            if (lane == 0) hs = atomicAdd(&p.ctrl->nhub_items, 1u);
                            hs = __shfl_sync(0xffffffffu, hs, 0);
                            if (hs < p.hitem_cap) {
                                hslot = (int)hs;
#pragma unroll
                                for (int k = 0; k < KGRP; ++k) p.hubF[((uint64_t)hs * KGRP + k) * 32 + lane] = f[k];
                                if (lane == 0) p.hitems[hs] = HubItem{(uint32_t)row, xw, (uint32_t)nk, bits};
                            }
                        }
                        if (hslot >= 0) {
                            // records of ~HUB_LOADS visited-word loads per lane: fewer
                            // edges per record when more chunks are active
                            const uint32_t seglen = hub_seglen(nk);
                            const uint32_t nseg = (end - beg + seglen - 1) / seglen;
                            uint32_t r = 0;
                            if (lane == 0) r = atomicAdd(&p.ctrl->nhub_recs, nseg);
                            r = __shfl_sync(0xffffffffu, r, 0);
                            if (r + nseg <= p.hrec_cap) {
                                for (uint32_t sg = lane; sg < nseg; sg += 32) {
                                    const uint32_t b0 = beg + sg * seglen;
                                    p.hrecs[r + sg] = HubRec{(uint32_t)hslot, (uint32_t)t, b0, min(end, b0 + seglen)};
                                }
                                continue;
                            }
                            for (uint32_t sg = lane; r + sg < p.hrec_cap && sg < nseg; sg += 32)
                                p.hrecs[r + sg] = HubRec{0u, 0u, 0u, 0u};
                        }
                    }
                    if constexpr (TMA) {
                        // chunk window of the group (bits ascend: chunk of k = 0 is the first)
                        const uint32_t c0 = (uint32_t)bits & 0xffu;
                        const uint32_t cl = (uint32_t)(bits >> (8 * (nk - 1))) & 0xffu;
                        const uint32_t span = cl - c0 + 1u;
                        if (nk >= 2 && span <= (uint32_t)KGRP && (xw * 32u + c0 + span) * 32u <= p.nw) {
                            expand_edges_tma<STATS>(p, S, A.tto[t], A.nbr[slot], beg, end, f, bits, nk, c0, span, xw,
                                                    lane, st, act, A.toff[A.tto[t] + 1] > A.toff[A.tto[t]], ring);
                            continue;
                        }
                    }
                    dispatch_edges<STATS, BND>(nk, p, S, A.tto[t], A.nbr[slot], beg, end, f, bits, xw, lane, st, act,
                                          A.toff[A.tto[t] + 1] > A.toff[A.tto[t]]);
                }
            }
        }
    }
    if (__ballot_sync(0xffffffffu, act) && lane == 0) p.ctrl->active[p.par ^ 1] = 1u;
    flush_stats<STATS>(st, p.stats);
    if (!TMA && p.pull_mode) act_flush(actS, p.ActNext, p.nw);
}

// Deferred long rows: a warp per HUB_EDGES-edge segment.
template <bool STATS, bool BND = false, bool TMA = false>
__global__ void __launch_bounds__(256, TMA ? RPQ_TMA_MINB : RPQ_HUB_MINB) k_level_hub(const DevAuto A,
                                                                                    const Layout *__restrict__ Sg,
                                                                                    const LevelArgs p) {
    if (BND && *(volatile const uint32_t *)&p.ctrl->blevel > p.level_lim) return;   // length bound reached
    __shared__ Layout S;
    extern __shared__ __align__(128) unsigned char tma_dyn[];
    load_layout(S, Sg, A.nq);
    const int lane = threadIdx.x & 31;
    TmaRing ring{};
    if constexpr (TMA) {
        unsigned char *wb = tma_dyn + (threadIdx.x >> 5) * TMA_WARP_BYTES;
        ring.bar = reinterpret_cast<uint64_t *>(wb);
        ring.buf = reinterpret_cast<uint64_t *>(wb + 64);
        if (lane == 0) {
            for (int sl = 0; sl < TMA_NS; ++sl) mbar_init(ring.bar + sl, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    const uint32_t n = min(p.ctrl->nhub_recs, p.hrec_cap);
    unsigned long long st[NSTAT] = {};
    bool act = false;
    (void)wid; (void)nwarps;
    // records differ in cost (1-8 chunks x up to HUB_EDGES edges): fetched
    // dynamically, one atomic per record
    for (;;) {
        uint32_t it = 0;
        if (lane == 0) it = atomicAdd(&p.ctrl->hcur, 1u);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= n) break;
        const HubRec r = p.hrecs[it];
        if (r.end == r.beg) continue;
        const HubItem h = p.hitems[r.hitem];
        uint64_t f[KGRP];
#pragma unroll
        for (int k = 0; k < KGRP; ++k) f[k] = p.hubF[((uint64_t)r.hitem * KGRP + k) * 32 + lane];
        if constexpr (TMA) {
            const int nk = (int)h.nk;
            const uint32_t c0 = (uint32_t)h.bits & 0xffu;
            const uint32_t span = ((uint32_t)(h.bits >> (8 * (nk - 1))) & 0xffu) - c0 + 1u;
            if (span <= (uint32_t)KGRP && (h.xw * 32u + c0 + span) * 32u <= p.nw) {
                expand_edges_tma<STATS>(p, S, A.tto[r.t], A.nbr[A.tslot[r.t]], r.beg, r.end, f, h.bits, nk, c0, span,
                                        h.xw, lane, st, act, A.toff[A.tto[r.t] + 1] > A.toff[A.tto[r.t]], ring);
                continue;
            }
        }
        dispatch_edges<STATS, BND>((int)h.nk, p, S, A.tto[r.t], A.nbr[A.tslot[r.t]], r.beg, r.end, f, h.bits, h.xw, lane,
                              st, act, A.toff[A.tto[r.t] + 1] > A.toff[A.tto[r.t]]);
    }
    if (__ballot_sync(0xffffffffu, act) && lane == 0) p.ctrl->active[p.par ^ 1] = 1u;
    flush_stats<STATS>(st, p.stats);
}

// ---- bottom-up (pull) levels: direction-optimising BFS --------
// A level whose active-unit fraction exceeds the threshold runs bottom-up:
// every (target row, 32-word chunk) with sources that are still active and
// have not reached it (need = Act & ~Vis) ORs the visited words of its
// in-neighbours (transposed CSR, entering transitions) until need is
// covered, then writes the new bits with a plain store -- one owner per
// word, no atomics, early exit once the row is complete (the dense levels of
// knows+, where most rows fill from their first in-neighbours).  Reading Vis
// (not the frontier) of the in-neighbours is exact: bits of Vis that are not
// in the frontier were already propagated along every out-edge.

// Before a pull level: consume the level's activity (X words -> TX) and mark
// every bit of the active chunks expanded (Done = Vis): the pull propagates
// all of Vis, so afterwards the frontier is exactly the new bits.
__global__ void k_pull_prep(const DevAuto A, const LevelArgs p) {
    if (!level_pull(p)) return;
    const int lane = threadIdx.x & 31;
    const uint32_t nunits = *(volatile uint32_t *)&p.ctrl->ucnt[p.par];
    for (;;) {
        uint32_t ui = 0;
        if (lane == 0) ui = atomicAdd(&p.ctrl->ucur[p.par], 1u);
        ui = __shfl_sync(0xffffffffu, ui, 0);
        if (ui >= nunits) break;
        const uint64_t u = p.ulist[ui];
        const uint64_t xi_l = u * 32 + lane;
        const uint32_t xl = xi_l < p.nxwords ? __ldcg(p.Xcur + xi_l) : 0u;
        bool fresh = false;
        if (xl) {
            p.Xcur[xi_l] = 0u;
            const uint32_t t0 = p.TX[xi_l];
            p.TX[xi_l] = t0 | xl;
            fresh = t0 == 0u;
        }
        {
            const unsigned fm = __ballot_sync(0xffffffffu, fresh);
            if (fm && lane == 0) atomicAdd(&p.ctrl->txw, (uint32_t)__popc(fm));
        }
        unsigned todo = __ballot_sync(0xffffffffu, xl != 0);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            uint32_t x = __shfl_sync(0xffffffffu, xl, src);
            const uint64_t xi = u * 32 + src;
            const uint64_t row = xi / p.nxw;
            const uint32_t xw = (uint32_t)(xi % p.nxw);
            while (x) {
                const uint32_t bt = (uint32_t)(__ffs(x) - 1);
                x &= x - 1;
                const uint64_t col = (uint64_t)(xw * 32u + bt) * 32u + lane;   // cw == 32
                if (col < p.nw) p.Done[row * p.nw + col] = ld_cg(p.Vis + row * p.nw + col);
            }
        }
    }
}

// OR of the in-neighbours' visited words of column col for target (q2, v),
// stopping as soon as every needed bit is covered (8 loads in flight).
template <bool STATS>
__device__ __forceinline__ uint64_t pull_gather(const DevAuto &A, const Layout &S, const LevelArgs &p, int q2,
                                                uint32_t v, uint32_t col, uint64_t need, int lane,
                                                unsigned long long *st, uint32_t *visited = nullptr) {
    const int it0 = A.itoff[q2], it1 = A.itoff[q2 + 1];
    uint64_t acc = 0;
    uint32_t nvis = 0;
    for (int it = it0; it < it1 && __any_sync(0xffffffffu, (need & ~acc) != 0); ++it) {
        const int q = A.itfrom[it], slot = A.itslot[it];
        const uint32_t beg = __ldg(A.ioff[slot] + v), end = __ldg(A.ioff[slot] + v + 1);
        const uint32_t lo = S.lo[q], len = S.len[q];
        const uint64_t tb = S.row_base[q] - lo;
        for (uint32_t j = beg; j < end; j += 32) {
            const uint32_t my = (j + lane < end) ? __ldg(A.inbr[slot] + j + lane) : 0u;
            const int cnt = (int)min(32u, end - j);
            bool done = false;
            for (int e0 = 0; e0 < cnt && !done; e0 += 8) {
                const bool want = (need & ~acc) != 0;
                uint64_t x[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const uint32_t u = __shfl_sync(0xffffffffu, my, (e0 + e) & 31);
                    const bool ok = want && e0 + e < cnt && u - lo < len;
                    x[e] = ok ? ld_cg(p.Vis + (tb + u) * p.nw + col) : 0ull;
                    if (STATS && ok) st[S_PULL_LOADS]++;
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) acc |= x[e];
                nvis += (uint32_t)min(8, cnt - e0);
                done = !__any_sync(0xffffffffu, (need & ~acc) != 0);
            }
            if (done) break;
        }
    }
    if (visited) *visited = nvis;
    return acc;
}

constexpr uint32_t PULL_TASKS = 32;   // (chunk, row) tasks per cursor fetch

template <bool STATS>
__global__ void __launch_bounds__(256) k_pull(const DevAuto A, const Layout *__restrict__ Sg, const LevelArgs p) {
    if (!level_pull(p)) return;
    __shared__ Layout S;
    __shared__ unsigned long long actS[ACT_SMEM_WORDS];
    load_layout(S, Sg, A.nq);
    act_init(actS, p.nw);
    const int lane = threadIdx.x & 31;
    const uint64_t nrows = S.row_base[A.nq - 1] + S.len[A.nq - 1];
    const uint32_t nch = p.nw / 32u;
    const uint64_t ntask = nrows * nch;
    unsigned long long st[NSTAT] = {};
    bool act = false;
    for (;;) {
        uint32_t t0 = 0;
        if (lane == 0) t0 = atomicAdd(&p.ctrl->pcur[p.par], PULL_TASKS);
        t0 = __shfl_sync(0xffffffffu, t0, 0);
        if (t0 >= ntask) break;
        const uint64_t t1 = ntask < (uint64_t)t0 + PULL_TASKS ? ntask : (uint64_t)t0 + PULL_TASKS;
        for (uint64_t t = t0; t < t1; ++t) {
            const uint32_t c = (uint32_t)(t / nrows);          // chunk-major: a run of rows per chunk
            const uint64_t row = t - (uint64_t)c * nrows;
            const int q2 = row_state(S, A.nq, row);
            const int it0 = A.itoff[q2], it1 = A.itoff[q2 + 1];
            if (it0 == it1) continue;                            // nothing enters q2
            const uint32_t col = c * 32u + lane;
            const uint64_t wi = row * p.nw + col;
            if (STATS && lane == 0) st[S_PULL_WORDS] += 32;
            const uint64_t vis = ld_cg(p.Vis + wi);
            const uint64_t need = ld_cg(p.ActCur + col) & ~vis;
            if (!__any_sync(0xffffffffu, need != 0)) continue;
            const uint32_t v = S.lo[q2] + (uint32_t)(row - S.row_base[q2]);
            const uint64_t acc = pull_gather<STATS>(A, S, p, q2, v, col, need, lane, st);
            const uint64_t nb = need & acc;
            if (nb) {
                p.Vis[wi] = vis | nb;                      // single owner of the word in a pull level
                act_or(actS, p.ActNext, col, nb);
            }
            if (__any_sync(0xffffffffu, nb != 0) && lane == 0 && A.toff[q2 + 1] > A.toff[q2]) {
                const uint64_t xi = row * p.nxw + c / 32u;
                red_or32(p.Xnext + xi, 1u << (c & 31u));
                red_or32(p.XBnext + (xi >> 10), 1u << ((xi >> 5) & 31));
                act = true;
            }
        }
    }
    if (__ballot_sync(0xffffffffu, act) && lane == 0) p.ctrl->active[p.par ^ 1] = 1u;
    if (STATS && threadIdx.x == 0 && blockIdx.x == 0) st[S_PULL_LEVELS] = 1;
    flush_stats<STATS>(st, p.stats);
    act_flush(actS, p.ActNext, p.nw);
}

// PE after the fact (RPQ_STATS; reading R12): sum over rows (q, v) of
// popcount(Vis) x product out-degree of (v, q).  Exact whatever the
// direction of each level (pull levels do not expand bits one by one).
__global__ void k_pe_rows(const DevAuto A, const Layout S, const uint64_t *Vis, uint32_t nw,
                          unsigned long long *out) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    const uint64_t nrows = S.row_base[A.nq - 1] + S.len[A.nq - 1];
    unsigned long long acc = 0;
    for (uint64_t row = wid; row < nrows; row += nwarps) {
        const int q = row_state(S, A.nq, row);
        if (A.toff[q + 1] == A.toff[q]) continue;
        const uint32_t v = S.lo[q] + (uint32_t)(row - S.row_base[q]);
        unsigned long long pc = 0;
        for (uint32_t w = lane; w < nw; w += 32) pc += __popcll(ld_cg(Vis + row * nw + w));
#pragma unroll
        for (int o = 16; o; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
        if (!pc) continue;
        unsigned long long deg = 0;
        for (int t = A.toff[q]; t < A.toff[q + 1]; ++t)
            deg += __ldg(A.off[A.tslot[t]] + v + 1) - __ldg(A.off[A.tslot[t]] + v);
        acc += pc * deg;
    }
    if (lane == 0 && acc) atomicAdd(out, acc);
}

// Per-source PE (RPQ_SOURCE_PE): pe[i] += sum over rows (q, v) with bit i in
// Vis of the product out-degree of (v, q).  A warp takes a tile of 32 rows x 4
// words: lane = row, and for every bit position the warp sums the out-degrees
// of the rows that have it with one REDUX (__reduce_add_sync); lane b keeps
// bits b and b + 32.  A verification mode (parity of the PE numerator per
// source), not on the timed path.
constexpr uint32_t SPE_TILES = 64;   // 32-row tiles per task (atomics amortised)
__global__ void k_source_pe(const DevAuto A, const Layout S, const uint64_t *Vis, uint32_t nw, uint32_t nb,
                            unsigned long long *pe) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    const uint64_t nrows = S.row_base[A.nq - 1] + S.len[A.nq - 1];
    const uint64_t ntiles = (nrows + 31) / 32, ngrp = (nw + 3) / 4;
    const uint64_t nchunks = (ntiles + SPE_TILES - 1) / SPE_TILES;
    for (uint64_t task = wid; task < nchunks * ngrp; task += nwarps) {
        const uint32_t w0 = (uint32_t)(task % ngrp) * 4;
        const uint64_t t0 = (task / ngrp) * SPE_TILES;
        unsigned long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint64_t t = t0; t < t0 + SPE_TILES && t < ntiles; ++t) {
            const uint64_t row = t * 32 + lane;
            uint32_t d = 0;
            if (row < nrows) {
                const int q = row_state(S, A.nq, row);
                d = prod_deg(A, q, S.lo[q] + (uint32_t)(row - S.row_base[q]));
            }
            if (!__any_sync(0xffffffffu, d != 0)) continue;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t x = (d && w0 + k < nw) ? ld_cg(Vis + row * nw + w0 + k) : 0ull;
                if (!__any_sync(0xffffffffu, x != 0)) continue;
#pragma unroll 8
                for (int b = 0; b < 32; ++b) {
                    const uint32_t s0 = __reduce_add_sync(0xffffffffu, ((x >> b) & 1ull) ? d : 0u);
                    const uint32_t s1 = __reduce_add_sync(0xffffffffu, ((x >> (b + 32)) & 1ull) ? d : 0u);
                    if (lane == b) { acc[2 * k] += s0; acc[2 * k + 1] += s1; }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i0 = (w0 + k) * 64 + lane, i1 = i0 + 32;
            if (acc[2 * k] && i0 < nb) atomicAdd(pe + i0, acc[2 * k]);
            if (acc[2 * k + 1] && i1 < nb) atomicAdd(pe + i1, acc[2 * k + 1]);
        }
    }
}

// per-source PE of the seeds when q0 has no rows: out-degree of (s_i, q0)
__global__ void k_source_pe_seeds(const DevAuto A, const uint32_t *cand, const uint32_t *pidx, uint64_t b0, uint32_t nb,
                                  unsigned long long *pe) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x)
        pe[i] += prod_deg(A, 0, cand[pidx[b0 + i]]);
}

// PE of the seeds when q0 has no rows (k_seed_expand): out-degree of (s, q0).
__global__ void k_pe_seeds(const DevAuto A, const uint32_t *cand, const uint32_t *pidx, uint64_t b0, uint32_t nb,
                           unsigned long long *out) {
    unsigned long long acc = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
        const uint32_t sv = cand[pidx[b0 + i]];
        for (int t = A.toff[0]; t < A.toff[1]; ++t)
            acc += __ldg(A.off[A.tslot[t]] + sv + 1) - __ldg(A.off[A.tslot[t]] + sv);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// Seed batch sources: source i of the batch gets bit i in N of row (q0, s_i)
// and its chunk is marked active; the first level moves it into Vis.  With
// `skip_q0` (q0 has no incoming transition and is not final, so its rows
// would only ever hold the seeds) nothing is written here: k_seed_expand
// expands the seeds directly and q0 gets no rows at all.
__global__ void k_seed(const Layout S, const uint32_t *__restrict__ cand, const uint32_t *__restrict__ pidx,
                       uint64_t b0, uint32_t nb, uint64_t *Vis, uint32_t *X, uint32_t *XB, uint32_t nw, uint32_t nxw,
                       uint32_t cw, Ctrl *ctrl, int skip_q0, uint64_t *act0) {
    // every batch source is active at the first level (pull filter)
    if (act0)
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x)
            atomicOr((unsigned long long *)act0 + (i >> 6), 1ull << (i & 63));
    if (!skip_q0)
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
            const uint32_t s = cand[pidx[b0 + i]];
            const uint64_t row = S.row_base[0] + (s - S.lo[0]);
            const uint32_t w = i >> 6, c = w / cw;
            Vis[row * nw + w] = 1ull << (i & 63);        // rows are distinct: plain stores
            const uint64_t xi = row * nxw + c / 32;
            X[xi] = 1u << (c & 31);
            atomicOr(XB + (xi >> 10), 1u << ((xi >> 5) & 31));
        }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctrl->active[0] = (nb && !skip_q0) ? 1u : 0u;
        ctrl->active[1] = 0;
        ctrl->nhub_items = 0;
        ctrl->nhub_recs = 0;
        ctrl->hcur = 0;
        ctrl->ucnt[0] = ctrl->ucnt[1] = 0;
        ctrl->ucur[0] = ctrl->ucur[1] = 0;
        ctrl->ntouched = 0;
        ctrl->blevel = 0;
        ctrl->txw = 0;
    }
}

// Level 0 without q0 rows, short seed rows: a THREAD per batch source ORs
// its single bit into every neighbour's visited word (and marks the target
// chunk active); one bit per source means the warp-per-source path below
// would keep 31 lanes idle (knows+: 65 K sources x ~61 edges took 2.6 ms).
// Rows with more than SEED_LANE_MAX edges stay with the warp path.  XB is
// set afterwards from X (k_xb_from_x) instead of one contended OR per edge.
constexpr uint32_t SEED_LANE_MAX = 256;
__global__ void __launch_bounds__(256) k_seed_lanes(const DevAuto A, const Layout *__restrict__ Sg,
                                                    const LevelArgs p, const uint32_t *__restrict__ cand,
                                                    const uint32_t *__restrict__ pidx, uint64_t b0, uint32_t nb) {
    __shared__ Layout S;
    load_layout(S, Sg, A.nq);
    bool act = false;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
        const uint32_t sv = cand[pidx[b0 + i]];
        const uint32_t w = i >> 6, c = w / p.cw;
        const uint64_t bit = 1ull << (i & 63);
        for (int t = A.toff[0]; t < A.toff[1]; ++t) {
            const int slot = A.tslot[t];
            const uint32_t beg = __ldg(A.off[slot] + sv), end = __ldg(A.off[slot] + sv + 1);
            if (end == beg || end - beg > SEED_LANE_MAX) continue;
            const uint32_t q2 = A.tto[t];
            const bool live2 = A.toff[q2 + 1] > A.toff[q2];
            const uint64_t tbase = S.row_base[q2] - S.lo[q2];
            for (uint32_t j = beg; j < end; ++j) {
                const uint64_t trow = tbase + __ldg(A.nbr[slot] + j);
                red_or64(p.Disc + trow * p.nw + w, bit);
                if (live2) {
                    red_or32(p.Xnext + trow * p.nxw + (c >> 5), 1u << (c & 31u));
                    act = true;
                }
            }
        }
    }
    if (__any_sync(0xffffffffu, act) && (threadIdx.x & 31) == 0) p.ctrl->active[p.par ^ 1] = 1u;
}

__global__ void k_xb_from_x(const uint32_t *X, uint64_t nxwords, uint32_t *XB) {
    for (uint64_t i0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull; i0 < nxwords;
         i0 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = i0 + (threadIdx.x & 31);
        const bool nz = i < nxwords && X[i] != 0u;
        if (__ballot_sync(0xffffffffu, nz) && (threadIdx.x & 31) == 0)
            atomicOr(XB + (i0 >> 10), 1u << ((i0 >> 5) & 31));
    }
}

// Level 0 without q0 rows: a warp per batch source expands its single bit
// along q0's transitions straight into N / X / XB of the parity-0 level.
// p must be the parity-1 argument set (its "next" buffers are parity 0).
template <bool STATS, bool BND = false>
__global__ void __launch_bounds__(256) k_seed_expand(const DevAuto A, const Layout *__restrict__ Sg,
                                                     const LevelArgs p, const uint32_t *__restrict__ cand,
                                                     const uint32_t *__restrict__ pidx, uint64_t b0, uint32_t nb,
                                                     int long_only) {
    __shared__ Layout S;
    load_layout(S, Sg, A.nq);
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    unsigned long long st[NSTAT] = {};
    bool act = false;
    for (uint64_t i = wid; i < nb; i += nwarps) {
        const uint32_t sv = cand[pidx[b0 + i]];
        const uint32_t w = (uint32_t)(i >> 6), c = w / p.cw;
        uint64_t f[KGRP] = {};
        if (lane == (int)(w - c * p.cw)) f[0] = 1ull << (i & 63);
        const uint64_t bits = c & 31u;
        const uint32_t xw = c >> 5;
        if (STATS && lane == 0) st[S_ITEMS]++;
        for (int t = A.toff[0]; t < A.toff[1]; ++t) {
            const int slot = A.tslot[t];
            const uint32_t beg = __ldg(A.off[slot] + sv), end = __ldg(A.off[slot] + sv + 1);
            if (STATS && lane == 0) st[S_ITEM_TRANS]++;
            if (long_only && end - beg <= SEED_LANE_MAX) continue;   // done by k_seed_lanes
            if (end - beg > HUB_EDGES) {
                // long seed row (e.g. a single target with 10^5 in-edges):
                // its HUB_EDGES segments go to k_level_hub, launched next
                uint32_t hs = 0;
                if (lane == 0) hs = atomicAdd(&p.ctrl->nhub_items, 1u);
                hs = __shfl_sync(0xffffffffu, hs, 0);
                const uint32_t nseg = (end - beg + HUB_EDGES - 1) / HUB_EDGES;
                uint32_t r = 0;
                if (hs < p.hitem_cap && lane == 0) r = atomicAdd(&p.ctrl->nhub_recs, nseg);
                r = __shfl_sync(0xffffffffu, r, 0);
                if (hs < p.hitem_cap && r + nseg <= p.hrec_cap) {
#pragma unroll
                    for (int k = 0; k < KGRP; ++k) p.hubF[((uint64_t)hs * KGRP + k) * 32 + lane] = f[k];
                    if (lane == 0) p.hitems[hs] = HubItem{0u, xw, 1u, bits};
                    for (uint32_t sg = lane; sg < nseg; sg += 32) {
                        const uint32_t s0 = beg + sg * HUB_EDGES;
                        p.hrecs[r + sg] = HubRec{hs, (uint32_t)t, s0, min(end, s0 + HUB_EDGES)};
                    }
                    continue;
                }
                if (hs < p.hitem_cap)   // records did not fit: neutralise the reserved ones
                    for (uint32_t sg = lane; r + sg < p.hrec_cap && sg < nseg; sg += 32)
                        p.hrecs[r + sg] = HubRec{0u, 0u, 0u, 0u};
            }
            if (end > beg)
                expand_edges<1, STATS, BND>(p, S, A.tto[t], A.nbr[slot], beg, end, f, bits, xw, lane, st, act,
                                       A.toff[A.tto[t] + 1] > A.toff[A.tto[t]]);
        }
    }
    if (__ballot_sync(0xffffffffu, act) && lane == 0) p.ctrl->active[p.par ^ 1] = 1u;
    flush_stats<STATS>(st, p.stats);
}

// ---- sparse engine ----------------------------------------------------------
// For queries whose per-source reach is small (replyOf* chains, selective
// atoms), a warp evaluates one source at a time: the product-graph BFS of
// P:252-257 with the visited set as an open-addressing hash set of (v, q)
// keys and the frontier as a FIFO, both in shared memory.  Distinct final
// targets are counted through marker keys (v, 255) in the same set.  A source
// whose reach outgrows the warp's capacity is flagged and re-evaluated by the
// dense bit-parallel engine.
constexpr int SP_WARPS = 4;
constexpr int SP_H = 1024;           // hash slots per warp (u64 keys)
constexpr int SP_Q = 512;            // FIFO capacity per warp
constexpr int SP_PROBES = 32;
constexpr uint64_t SP_EMPTY = ~0ull;

__device__ __forceinline__ int sp_insert(uint64_t *tab, uint64_t key) {
    uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 54);   // 10 bits
    for (int pr = 0; pr < SP_PROBES; ++pr) {
        const uint64_t old = atomicCAS((unsigned long long *)&tab[h], (unsigned long long)SP_EMPTY,
                                       (unsigned long long)key);
        if (old == SP_EMPTY) return 1;
        if (old == key) return 0;
        h = (h + 1) & (SP_H - 1);
    }
    return -1;
}

// idx == nullptr: productive indices [0, np) restricted to this shard's
// batches (batch = i / B); else the n listed productive indices.
// WRITE: second pass of PAIRS mode -- re-run the BFS of every source that
// did not overflow and write its distinct targets, sorted, at start[cand].
template <bool STATS, bool WRITE>
__global__ void __launch_bounds__(SP_WARPS * 32) k_sparse(const DevAuto A, const uint32_t *__restrict__ cand,
                                                          const uint32_t *__restrict__ pidx,
                                                          const uint32_t *__restrict__ idx, uint64_t n, uint64_t B,
                                                          uint32_t shard_index, uint32_t shard_count,
                                                          unsigned long long *counts, uint8_t *overflow,
                                                          unsigned long long *stats,
                                                          const unsigned long long *start = nullptr,
                                                          uint32_t *osrc = nullptr, uint32_t *odst = nullptr,
                                                          int *err = nullptr, const uint64_t *n_dev = nullptr,
                                                          unsigned long long *spe = nullptr) {
    __shared__ uint64_t tab_s[SP_WARPS][SP_H];
    if (n_dev) n = *n_dev;
    __shared__ uint64_t que_s[SP_WARPS][SP_Q];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    uint64_t *tab = tab_s[wl], *que = que_s[wl];
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    unsigned long long pe_acc = 0, src_done = 0;
    for (uint64_t it = wid; it < n; it += nwarps) {
        const uint64_t pi = idx ? idx[it] : it;
        if (!idx && (pi / B) % shard_count != shard_index) continue;
        if (WRITE && overflow[pi]) continue;
        const uint32_t s = cand[pidx[pi]];
        for (int k = lane; k < SP_H; k += 32) tab[k] = SP_EMPTY;
        __syncwarp();
        unsigned long long cnt = 0, pe = 0;
        bool ovf = false;
        int head = 0, tail = 1;
        if (lane == 0) {
            sp_insert(tab, (uint64_t)s << 8);
            que[0] = (uint64_t)s << 8;
            if (A.final_mask & 1ull) { sp_insert(tab, ((uint64_t)s << 8) | 255u); cnt = 1; }
        }
        __syncwarp();
        while (head < tail && !ovf) {
            const uint64_t key = que[head++];
            const uint32_t v = (uint32_t)(key >> 8), q = (uint32_t)(key & 0xff);
            for (int t = A.toff[q]; t < A.toff[q + 1] && !ovf; ++t) {
                const uint32_t q2 = A.tto[t];
                const bool fin2 = (A.final_mask >> q2) & 1ull;
                const bool live2 = A.toff[q2 + 1] > A.toff[q2];
                const uint32_t *off = A.off[A.tslot[t]];
                const uint32_t beg = __ldg(off + v), end = __ldg(off + v + 1);
                pe += end - beg;
                const uint32_t *nbr = A.nbr[A.tslot[t]];
                for (uint32_t j = beg; j < end && !ovf; j += 32) {
                    const bool valid = j + lane < end;
                    const uint32_t w = valid ? __ldg(nbr + j + lane) : 0u;
                    const int ins = valid ? sp_insert(tab, ((uint64_t)w << 8) | q2) : 0;
                    if (__ballot_sync(0xffffffffu, ins < 0)) { ovf = true; break; }
                    const unsigned newm = __ballot_sync(0xffffffffu, ins == 1);
                    if (live2 && newm) {
                        const int pos = tail + __popc(newm & lt);
                        if (ins == 1 && pos < SP_Q) que[pos] = ((uint64_t)w << 8) | q2;
                        tail += __popc(newm);
                        if (tail > SP_Q) { ovf = true; break; }
                    }
                    if (fin2 && newm) {
                        const int r2 = (ins == 1) ? sp_insert(tab, ((uint64_t)w << 8) | 255u) : 0;
                        if (__ballot_sync(0xffffffffu, r2 < 0)) { ovf = true; break; }
                        cnt += __popc(__ballot_sync(0xffffffffu, r2 == 1));
                    }
                }
                __syncwarp();
            }
        }
        if constexpr (WRITE) {
            if (ovf) {   // the first pass fitted; a different probe order did not
                if (lane == 0) atomicExch(err, 1);
                continue;
            }
            // gather the target markers (v, 255) and write them ranked
            uint32_t *lst = reinterpret_cast<uint32_t *>(que);
            int nl = 0;
            for (int k0 = 0; k0 < SP_H; k0 += 32) {
                const uint64_t key = tab[k0 + lane];
                const bool mk = key != SP_EMPTY && (key & 0xff) == 255u;
                const unsigned mm = __ballot_sync(0xffffffffu, mk);
                if (mk) lst[nl + __popc(mm & lt)] = (uint32_t)(key >> 8);
                nl += __popc(mm);
            }
            __syncwarp();
            const unsigned long long base = start[pidx[pi]];
            for (int i = lane; i < nl; i += 32) {
                const uint32_t t = lst[i];
                int r = 0;
                for (int j = 0; j < nl; ++j) r += lst[j] < t;
                osrc[base + r] = s;
                odst[base + r] = t;
            }
            __syncwarp();
        } else {
            if (lane == 0) {
                counts[pi] = ovf ? 0ull : cnt;
                overflow[pi] = ovf ? 1 : 0;
                if (spe) spe[pi] = ovf ? 0ull : pe;
            }
            if (!ovf) { pe_acc += pe; src_done++; }
        }
        __syncwarp();
    }
    if (STATS && !WRITE && lane == 0) {
        if (pe_acc) atomicAdd(stats + S_PE, pe_acc);
        if (src_done) atomicAdd(stats + S_ITEMS, src_done);
    }
}

// Thread tier of the sparse engine: one thread per source, its visited
// (vertex, state) keys in a list of ST_K entries that is also the BFS FIFO
// (keys are appended in discovery order and expanded in that order).  Meant
// for reach sets of a handful of product vertices (replyOf* ancestor chains:
// depth ~2); a source that discovers more than ST_K keys or scans more than
// ST_EMAX edges is flagged (tovf) and goes to the warp tier (k_sparse).
// Distinct final targets are the distinct vertices of keys in final states.
constexpr int ST_K = 32;
constexpr uint32_t ST_EMAX = 256;

template <bool STATS, bool WRITE>
__global__ void __launch_bounds__(256) k_sparse_thread(const DevAuto A, const uint32_t *__restrict__ cand,
                                                       const uint32_t *__restrict__ pidx, uint64_t n, uint64_t B,
                                                       uint32_t shard_index, uint32_t shard_count,
                                                       unsigned long long *counts, uint8_t *tovf,
                                                       unsigned long long *stats,
                                                       const unsigned long long *start = nullptr,
                                                       uint32_t *osrc = nullptr, uint32_t *odst = nullptr,
                                                       unsigned long long *spe = nullptr) {
    uint64_t lst[ST_K];
    unsigned long long pe_acc = 0, src_done = 0;
    for (uint64_t pi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; pi < n;
         pi += (uint64_t)gridDim.x * blockDim.x) {
        if ((pi / B) % shard_count != shard_index) continue;
        if (WRITE && tovf[pi]) continue;
        const uint32_t s = cand[pidx[pi]];
        int nl = 1;
        lst[0] = (uint64_t)s << 8;
        bool ovf = false;
        uint32_t scanned = 0;
        for (int h = 0; h < nl && !ovf; ++h) {
            const uint32_t v = (uint32_t)(lst[h] >> 8), q = (uint32_t)(lst[h] & 0xff);
            for (int t = A.toff[q]; t < A.toff[q + 1] && !ovf; ++t) {
                const uint32_t q2 = A.tto[t];
                const uint32_t *off = A.off[A.tslot[t]];
                const uint32_t beg = __ldg(off + v), end = __ldg(off + v + 1);
                scanned += end - beg;
                if (scanned > ST_EMAX) { ovf = true; break; }
                const uint32_t *nbr = A.nbr[A.tslot[t]];
                for (uint32_t j = beg; j < end; ++j) {
                    const uint64_t key = ((uint64_t)__ldg(nbr + j) << 8) | q2;
                    bool found = false;
                    for (int i = 0; i < nl && !found; ++i) found = lst[i] == key;
                    if (found) continue;
                    if (nl == ST_K) { ovf = true; break; }
                    lst[nl++] = key;
                }
            }
        }
        if (ovf) {
            if (!WRITE) { tovf[pi] = 1; counts[pi] = 0; }
            continue;
        }
        // distinct vertices among keys in final states (first occurrences)
        unsigned long long cnt = 0;
        for (int i = 0; i < nl; ++i) {
            const uint32_t vi = (uint32_t)(lst[i] >> 8);
            if (!((A.final_mask >> (lst[i] & 0xff)) & 1ull)) continue;
            bool dup = false;
            for (int j = 0; j < i && !dup; ++j)
                dup = ((A.final_mask >> (lst[j] & 0xff)) & 1ull) && (uint32_t)(lst[j] >> 8) == vi;
            if (dup) continue;
            if constexpr (WRITE) {
                // rank among the distinct final vertices -> sorted output
                unsigned long long r = 0;
                for (int j = 0; j < nl; ++j) {
                    const uint32_t vj = (uint32_t)(lst[j] >> 8);
                    if (!((A.final_mask >> (lst[j] & 0xff)) & 1ull) || vj >= vi) continue;
                    bool dj = false;   // count each smaller vertex once
                    for (int k = 0; k < j && !dj; ++k)
                        dj = ((A.final_mask >> (lst[k] & 0xff)) & 1ull) && (uint32_t)(lst[k] >> 8) == vj;
                    r += !dj;
                }
                const unsigned long long o = start[pidx[pi]] + r;
                osrc[o] = s;
                odst[o] = vi;
            }
            ++cnt;
        }
        if (!WRITE) {
            counts[pi] = cnt;
            if (spe) spe[pi] = scanned;   // every reached key was expanded: its product edges (R12)
            if (STATS) {
                pe_acc += scanned;   // every key was expanded: the product edges of the reach (PE, R12)
                src_done++;
            }
        }
    }
    if (STATS && !WRITE) {
        if (pe_acc) atomicAdd(stats + S_PE, pe_acc);
        if (src_done) atomicAdd(stats + S_ITEMS, src_done);
    }
}

__global__ void k_sum_flags(const uint8_t *flag, const uint32_t *idx, uint64_t n, unsigned long long *out) {
    unsigned long long c = 0;
    for (uint64_t k = threadIdx.x; k < n; k += blockDim.x) c += flag[idx[k]];
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned long long w[32];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += w[i];
        *out = t;
    }
}

__global__ void k_gather_idx(const uint32_t *cand, const uint32_t *pidx, const uint32_t *list, uint64_t n,
                             uint32_t *out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = cand[pidx[list[i]]];
}

// per-candidate counts from the sparse pass (non-overflowed sources)
__global__ void k_sparse_scatter(const uint32_t *pidx, const unsigned long long *counts, const uint8_t *overflow,
                                 uint64_t np, uint64_t B, uint32_t shard_index, uint32_t shard_count,
                                 unsigned long long *cand_cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < np; i += (uint64_t)gridDim.x * blockDim.x)
        if ((i / B) % shard_count == shard_index && !overflow[i]) cand_cnt[pidx[i]] = counts[i];
}

// pairs of a dense sub-evaluation (sorted by source; sstart = scan of its
// per-source counts) copied to their places in the sparse PAIRS output
__global__ void k_place_sub(const uint32_t *cand, uint64_t nsrc, const uint32_t *ps_src,
                            const unsigned long long *ps_cnt, const unsigned long long *sstart, uint64_t n,
                            const uint32_t *ssrc, const uint32_t *sdst, const unsigned long long *start,
                            uint32_t *osrc, uint32_t *odst) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    for (uint64_t i = wid; i < n; i += nwarps) {
        uint64_t lo = 0, hi = nsrc;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (cand[mid] < ps_src[i]) lo = mid + 1; else hi = mid;
        }
        const unsigned long long o = start[lo], a = sstart[i], c = ps_cnt[i];
        for (unsigned long long k = lane; k < c; k += 32) {
            osrc[o + k] = ssrc[a + k];
            odst[o + k] = sdst[a + k];
        }
    }
}

// per-candidate counts of a dense sub-evaluation (source ids -> candidate
// indices by binary search in the sorted candidate list)
__global__ void k_scatter_sub(const uint32_t *cand, uint64_t nsrc, const uint32_t *src, const unsigned long long *c,
                              uint64_t n, unsigned long long *cand_cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = nsrc;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (cand[mid] < src[i]) lo = mid + 1; else hi = mid;
        }
        cand_cnt[lo] = c[i];
    }
}

// ---- productive sources: s with an out-edge under a label leaving q0 ------
__global__ void k_productive(const DevAuto A, const uint32_t *__restrict__ cand, uint64_t n, uint8_t *flag) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = cand[j];
        uint8_t f = 0;
        for (int t = A.toff[0]; t < A.toff[1] && !f; ++t) {
            const uint32_t *off = A.off[A.tslot[t]];
            f = __ldg(off + s + 1) > __ldg(off + s);
        }
        flag[j] = f;
    }
}

// per batch: first/last productive candidate index and their vertex ids
__global__ void k_batch_bounds(const uint32_t *pidx, const uint32_t *cand, uint64_t np, uint64_t B, uint64_t nbatches,
                               uint32_t *out) {
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nbatches; b += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t f = pidx[b * B], l = pidx[min(np, (b + 1) * B) - 1];
        out[4 * b + 0] = f;
        out[4 * b + 1] = l;
        out[4 * b + 2] = cand[f];
        out[4 * b + 3] = cand[l];
    }
}

// Dense clear of the batch state, only when the finished batch touched a
// large fraction of it (device-side decision: no host round trip).
__global__ void k_clear_dense(uint64_t *Vis, uint64_t *Done, uint64_t words, uint32_t *TX, uint64_t nxwords,
                              uint32_t *TU, uint64_t ntu, const Ctrl *ctrl, uint64_t nunits, int force_dense) {
    if (!force_dense && sparse_batch(ctrl, nunits, nxwords - 32)) return;
    const uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = i0; i < words; i += st) { Vis[i] = 0; Done[i] = 0; }
    for (uint64_t i = i0; i < nxwords; i += st) TX[i] = 0;
    for (uint64_t i = i0; i < ntu; i += st) TU[i] = 0;
}

// Length-bounded evaluation ends with the last level's discoveries (depth =
// the bound) still in N: fold both N arrays into Vis and zero them.
__global__ void k_merge_bounded(uint64_t *Vis, uint64_t *N0, uint64_t *N1, uint64_t words) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = N0[i], b = N1[i];
        if (a | b) {
            Vis[i] |= a | b;
            N0[i] = 0;
            N1[i] = 0;
        }
    }
}

__global__ void k_add_const(uint32_t *x, uint64_t n, uint32_t c) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
        x[j] += c;
}

__global__ void k_sample_idx(uint32_t *idx, uint64_t ns, uint64_t np) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < ns; k += (uint64_t)gridDim.x * blockDim.x)
        idx[k] = (uint32_t)(k * np / ns);
}

__global__ void k_prod_bounds(const uint64_t *d_np, const uint32_t *pidx, const uint32_t *cand, uint64_t *out) {
    if (threadIdx.x) return;
    const uint64_t np = *d_np;
    out[0] = np;
    out[1] = np ? cand[pidx[0]] : 0u;
    out[2] = np ? cand[pidx[np - 1]] : 0u;
}

__global__ void k_gather_u64(const unsigned long long *src, const uint64_t *idx, uint64_t n,
                             unsigned long long *out) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
        out[j] = src[idx[j]];
}

__global__ void k_iota(uint32_t *x, uint64_t n) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
        x[j] = (uint32_t)j;
}

// ---- extraction ------------------------------------------------------------
// Ans(v, w) = OR over final states q with v in range_q of Vis[row(q,v), w]:
// OR-ing the final states deduplicates targets reached in several final
// states (distinct pairs).
template <bool L1 = false>
__device__ __forceinline__ uint64_t ans_word(const DevAuto &A, const Layout &S, const uint64_t *Vis,
                                             uint32_t v, uint64_t w, uint32_t nw) {
    uint64_t acc = 0;
    uint64_t fm = A.final_mask;
    while (fm) {
        const int q = __ffsll((long long)fm) - 1;
        fm &= fm - 1;
        if (v - S.lo[q] < S.len[q]) {
            const uint64_t *p = Vis + (S.row_base[q] + (v - S.lo[q])) * nw + w;
            acc |= L1 ? __ldg((const unsigned long long *)p) : ld_cg(p);
        }
    }
    return acc;
}

// COUNT: total popcount of Ans over the hull [vlo, vlo + vn) x [0, nw).
// A warp per vertex row: lanes over the row's words (coalesced), 4 words per
// lane and final state loaded together so that every warp keeps several
// sectors in flight (a streaming read of the final states' rows).
// PE variant (pe != nullptr, RPQ_PE / RPQ_STATS): every state's row of v is
// read once -- final rows for the count, rows with product out-degree for
// popcount x out-degree -- so PE costs no extra pass when all states are
// final (e.g. (a|b)*c*).  [vlo, vlo + vn) must then cover every state's range.
__global__ void k_count_total(const DevAuto A, const Layout S, const uint64_t *Vis, uint32_t vlo, uint64_t vn,
                              uint32_t nw, unsigned long long *total, const Ctrl *ctrl, uint64_t nunits,
                              uint64_t nxwords, int force_dense, unsigned long long *pe = nullptr) {
    if (!force_dense && ctrl && sparse_batch(ctrl, nunits, nxwords)) return;   // sparse: k_count_touched counts
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    unsigned long long acc = 0, pacc = 0;
    const uint64_t qmask = pe ? ((A.nq >= 64 ? ~0ull : ((1ull << A.nq) - 1ull))) : A.final_mask;
    for (uint64_t r = wid; r < vn; r += nwarps) {
        const uint32_t v = vlo + (uint32_t)r;
        for (uint32_t w0 = 0; w0 < nw; w0 += 128) {
            uint64_t x[4] = {0, 0, 0, 0};
            uint64_t qm = qmask;
            while (qm) {
                const int q = __ffsll((long long)qm) - 1;
                qm &= qm - 1;
                if (v - S.lo[q] >= S.len[q]) continue;
                const bool fin = (A.final_mask >> q) & 1ull;
                const uint32_t d = pe ? prod_deg(A, q, v) : 0u;   // offsets: L1 hits after the first pass
                if (!fin && !d) continue;
                const uint64_t *rp = Vis + (S.row_base[q] + (v - S.lo[q])) * nw;
                uint64_t y[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t w = w0 + 32u * j + lane;
                    y[j] = w < nw ? ld_cg(rp + w) : 0ull;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (fin) x[j] |= y[j];
                    pacc += (unsigned long long)__popcll(y[j]) * d;
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) acc += __popcll(x[j]);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        pacc += __shfl_xor_sync(0xffffffffu, pacc, o);
    }
    if (lane == 0 && acc) atomicAdd(total, acc);
    if (lane == 0 && pacc) atomicAdd(pe, pacc);
}

// 32 x 32 bit-matrix transpose across a warp: lane i holds row i (bit j =
// element (i, j)); afterwards lane j holds column j (bit i = element (i, j)).
// Five rounds swap the off-diagonal s x s blocks (s = 16, 8, 4, 2, 1).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
    const uint32_t M[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const int sft = 16 >> r;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, sft);
        x = (lane & sft) ? ((x & ~M[r]) | ((y & ~M[r]) >> sft)) : ((x & M[r]) | ((y & M[r]) << sft));
    }
    return x;
}

// Per-(source, tile) counts by warp bit transposes.  Same task shape and
// coalesced sector loads as k_write_pairs (below): a CTA of 4 warps takes a
// group of 4 words (256 sources) and a part of tpp tiles of TILE_V vertices;
// the 512 x 4 visited words of a tile (OR over the final states) are staged
// in shared memory and warp w counts, per 32-vertex block of its word, the
// members of each source (lane b after the transpose: sources 64 w + b and
// + 32).  cnt[i * nseg + seg] (u32), i = batch-local source index.
constexpr int TC_XLD = TILE_V + 8;           // words k, k+1 in disjoint bank halves
__global__ void __launch_bounds__(128) k_tile_counts(const DevAuto A, const Layout S, const uint64_t *Vis, uint32_t vlo,
                                                     uint64_t vn, uint32_t nw, uint32_t nb, uint32_t nseg, uint32_t tpp,
                                                     uint32_t *cnt) {
    __shared__ __align__(16) uint64_t xs[4][TC_XLD];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const uint32_t k = threadIdx.x & 3u, r = threadIdx.x >> 2;
    const uint64_t nwg = (nw + 3) / 4;
    const uint64_t nparts = (nseg + tpp - 1) / tpp;
    for (uint64_t ct = blockIdx.x; ct < nwg * nparts; ct += gridDim.x) {
        const uint32_t g = (uint32_t)(ct % nwg);
        const uint32_t s0 = (uint32_t)(ct / nwg) * tpp, s1 = min(nseg, s0 + tpp);
        const uint32_t w = g * 4 + (uint32_t)wl, wk = g * 4 + k;
        for (uint32_t seg = s0; seg < s1; ++seg) {
            const uint64_t vbeg = (uint64_t)seg * TILE_V, vend = (vn < vbeg + TILE_V ? vn : vbeg + TILE_V);
            uint64_t xv[TILE_V / 32];
#pragma unroll
            for (int i = 0; i < TILE_V / 32; ++i) xv[i] = 0ull;
            uint64_t fm = wk < nw ? A.final_mask : 0ull;
            while (fm) {
                const int q = __ffsll((long long)fm) - 1;
                fm &= fm - 1;
                const uint32_t qlo = S.lo[q], qlen = S.len[q];
                const uint64_t qb = S.row_base[q];
#pragma unroll
                for (int i = 0; i < TILE_V / 32; ++i) {
                    const uint64_t vv = vbeg + r + 32u * (uint32_t)i;
                    const uint32_t d = vlo + (uint32_t)vv - qlo;
                    if (vv < vend && d < qlen) xv[i] |= ld_cg(Vis + (qb + d) * nw + wk);
                }
            }
            __syncthreads();                     // the previous tile's rows are consumed
#pragma unroll
            for (int i = 0; i < TILE_V / 32; ++i) xs[k][r + 32u * (uint32_t)i] = xv[i];
            __syncthreads();
            uint32_t c_lo = 0, c_hi = 0;
#pragma unroll
            for (int blk = 0; blk < TILE_V / 32; ++blk) {
                const uint64_t x = xs[wl][blk * 32 + lane];
                if (!__ballot_sync(0xffffffffu, x != 0)) continue;
                c_lo += __popc(warp_transpose32((uint32_t)x, lane));
                c_hi += __popc(warp_transpose32((uint32_t)(x >> 32), lane));
            }
            const uint32_t i0 = w * 64 + (uint32_t)lane, i1 = i0 + 32;
            if (w < nw && i0 < nb) cnt[(uint64_t)i0 * nseg + seg] = c_lo;
            if (w < nw && i1 < nb) cnt[(uint64_t)i1 * nseg + seg] = c_hi;
        }
    }
}

// Row-wise exclusive scan of cnt[i][0..nseg) (in place) -> row totals tot[i].
__global__ void k_row_scan(uint32_t *cnt, uint32_t nb, uint32_t nseg, unsigned long long *tot) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    for (uint64_t i = wid; i < nb; i += nwarps) {
        uint32_t *row = cnt + i * nseg;
        unsigned long long run = 0;
        for (uint32_t s0 = 0; s0 < nseg; s0 += 32) {
            const uint32_t s = s0 + lane;
            const uint32_t x = s < nseg ? row[s] : 0;
            uint32_t incl = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (s < nseg) row[s] = (uint32_t)run + incl - x;   // row offsets fit u32 (<= |V|)
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) tot[i] = run;
    }
}

// scatter productive row totals into the per-candidate count array
__global__ void k_scatter_counts(const unsigned long long *tot, const uint32_t *pidx, uint64_t b0, uint32_t nb,
                                 unsigned long long *cand_cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x)
        cand_cnt[pidx[b0 + i]] = tot[i];
}

__global__ void k_ps_flags(const unsigned long long *cnt, const unsigned long long *pe, uint64_t n, uint8_t *flag) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
        flag[j] = cnt[j] != 0 || (pe && pe[j] != 0);
}

__global__ void k_fill_eps(unsigned long long *cand_cnt, uint64_t n, unsigned long long val) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
        cand_cnt[j] = val;
}

constexpr int WP_WARPS = 4;
constexpr int WP_BLK = TILE_V / 32;          // 32-vertex blocks per tile
constexpr int WP_LD = WP_BLK + 1;            // padded row of masks (no bank conflicts)
// Write sorted (src, dst) pairs.  A CTA (4 warps) takes a group of 4
// consecutive words (256 sources) and a PART of tpp consecutive tiles, and
// walks the part tile by tile with each source's output offset kept in a
// register, so a source's whole part is ONE contiguous run written by one
// warp in order (no partial sectors between tiles).  Per tile:
//   (1) the CTA loads the 512 x 4 visited words (OR over the final states)
//       with each 32-byte row sector fetched by 4 adjacent lanes of one
//       request (a warp reading one word of 32 rows used 8 of 32 bytes
//       per sector) into shared memory;
//   (2) warp w transposes ITS word's row (bit transposes give, per source,
//       the masks of the tile's 32-vertex blocks) and keeps the masks in
//       place of that row (padded rows, conflict-free);
//   (3) per source, block by block, the lanes with a set bit write their
//       vertex to base + rank (rank = popcount of the lower lanes' bits) of
//       a per-warp staging buffer (consecutive words: no bank conflicts),
//       and ONE TMA bulk store (cp.async.bulk shared -> global) writes the
//       16-B-aligned body of the run; two buffers per warp, so the next
//       source is staged while the store drains.  Per-block global stores
//       instead serialised on the store address registers.  The source
//       column is a run of one value (16-byte vector stores).
// Offsets: start of the candidate + exclusive per-tile scan at the part's
// first tile, then + the source's count of every tile.
constexpr int WP3_XLD = TILE_V + 40;         // xs row: words k, k+1 in disjoint bank halves; holds 64 x WP_LD masks
__device__ __forceinline__ int wp_swz(int b, int blk) { return b * WP_LD + blk; }   // padded rows: conflict-free, immediate offsets
static_assert(WP3_XLD * 8 >= 64 * WP_LD * 4 && (WP3_XLD * 2) % 32 == 16, "xs row layout");
// TMA bulk store (smem -> global, 16-B aligned, size a multiple of 16) and its
// completion group (waiting for .read only frees the shared-memory source)
__device__ __forceinline__ void bulk_s2g(void *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
constexpr int WP_STG = TILE_V + 8;            // staging buffer of one source's tile run (u32, 16-B multiple)

__global__ void __launch_bounds__(WP_WARPS * 32, 6)
k_write_pairs(const DevAuto A, const Layout S, const uint64_t *Vis, uint32_t vlo, uint64_t vn, uint32_t nw,
               uint32_t nb, uint32_t nseg, uint32_t tpp, const uint32_t *cnt_scan, const uint32_t *cand,
               const uint32_t *pidx, uint64_t b0, const unsigned long long *start, uint64_t jlo, uint32_t *osrc,
               uint32_t *odst) {
    __shared__ __align__(16) uint64_t xs[4][WP3_XLD];
    __shared__ __align__(16) uint32_t stage_s[WP_WARPS][2][WP_STG];
    __shared__ uint32_t carry_s[WP_WARPS][64][8];                  // < 8 carried targets per source
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    int sbuf = 0;                                                  // staging buffer of the next source
    const int t = (int)threadIdx.x;
    const uint32_t lt = (1u << lane) - 1u;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(osrc) | reinterpret_cast<uintptr_t>(odst)) & 15u) == 0;
    const uint64_t nwg = (nw + 3) / 4;
    const uint64_t nparts = (nseg + tpp - 1) / tpp;
    const uint32_t k = (uint32_t)t & 3u, r = (uint32_t)t >> 2;    // this thread's word / first vertex of a tile
    for (uint64_t ct = blockIdx.x; ct < nwg * nparts; ct += gridDim.x) {
        // word-group-minor: concurrently running CTAs read neighbouring
        // sectors of the same rows
        const uint32_t g = (uint32_t)(ct % nwg);
        const uint32_t s0 = (uint32_t)(ct / nwg) * tpp, s1 = min(nseg, s0 + tpp);
        const uint32_t w = g * 4 + (uint32_t)wl, wk = g * 4 + k;
        unsigned long long o_lo = 0, o_hi = 0;
        uint32_t sid_lo = 0, sid_hi = 0, cc_lo = 0, cc_hi = 0;
        {
            const uint32_t i0 = w * 64 + (uint32_t)lane, i1 = i0 + 32;
            if (w < nw && i0 < nb) {
                const uint32_t j = pidx[b0 + i0];
                o_lo = start[j - jlo] + cnt_scan[(uint64_t)i0 * nseg + s0];
                sid_lo = cand[j];
            }
            if (w < nw && i1 < nb) {
                const uint32_t j = pidx[b0 + i1];
                o_hi = start[j - jlo] + cnt_scan[(uint64_t)i1 * nseg + s0];
                sid_hi = cand[j];
            }
        }
        for (uint32_t seg = s0; seg < s1; ++seg) {
            const uint64_t vbeg = (uint64_t)seg * TILE_V;
            {
                const uint64_t vend = (vn < vbeg + TILE_V ? vn : vbeg + TILE_V);
                uint64_t xv[WP_BLK];
#pragma unroll
                for (int i = 0; i < WP_BLK; ++i) xv[i] = 0ull;
                uint64_t fm = wk < nw ? A.final_mask : 0ull;
                while (fm) {
                    const int q = __ffsll((long long)fm) - 1;
                    fm &= fm - 1;
                    const uint32_t qlo = S.lo[q], qlen = S.len[q];
                    const uint64_t qb = S.row_base[q];
#pragma unroll
                    for (int i = 0; i < WP_BLK; ++i) {
                        const uint64_t vv = vbeg + r + 32u * (uint32_t)i;
                        const uint32_t d = vlo + (uint32_t)vv - qlo;
                        if (vv < vend && d < qlen) xv[i] |= ld_cg(Vis + (qb + d) * nw + wk);
                    }
                }
                __syncthreads();                 // every warp is done with the previous tile's masks
#pragma unroll
                for (int i = 0; i < WP_BLK; ++i) xs[k][r + 32u * (uint32_t)i] = xv[i];
                __syncthreads();
            }
            // (2) this warp's word row -> per-source block masks, in place
            uint64_t xr[WP_BLK];
#pragma unroll
            for (int blk = 0; blk < WP_BLK; ++blk) xr[blk] = xs[wl][blk * 32 + lane];
            __syncwarp();
            uint32_t *masks = reinterpret_cast<uint32_t *>(&xs[wl][0]);
#pragma unroll
            for (int blk = 0; blk < WP_BLK; ++blk) {
                masks[wp_swz(lane, blk)] = warp_transpose32((uint32_t)xr[blk], lane);
                masks[wp_swz(lane + 32, blk)] = warp_transpose32((uint32_t)(xr[blk] >> 32), lane);
            }
            __syncwarp();
            if (w >= nw) continue;
            // (3) per source of the warp's word.  Only whole 32-byte sectors
            // are written before the part's last tile: the < 8 trailing
            // targets of a tile run are carried (shared memory) to the next
            // tile's run of the same source, so no sector is written in two
            // halves far apart in time (L2 evicted such halves and HBM did a
            // read-modify-write: ~4 GB of extra reads per cfg2 a* launch).
            const bool last = seg + 1 == s1;
            const uint32_t vb = vlo + (uint32_t)vbeg + (uint32_t)lane;
            for (int b = 0; b < 64; ++b) {
                const uint32_t i = w * 64 + (uint32_t)b;
                if (i >= nb) break;
                // o = global index of the source's first unwritten (carried) target
                const unsigned long long o = __shfl_sync(0xffffffffu, b < 32 ? o_lo : o_hi, b & 31);
                const uint32_t cc = __shfl_sync(0xffffffffu, b < 32 ? cc_lo : cc_hi, b & 31);
                uint32_t *stg = stage_s[wl][sbuf];
                uint32_t *cry = carry_s[wl][b];
                const uint32_t off = (uint32_t)(o & 3ull);     // staged at (o mod 4): 16-B-aligned body
                if (lane == 0) bulk_wait_read<1>();            // the bulk store that last read this buffer is done
                __syncwarp();
                if ((uint32_t)lane < cc) stg[off + lane] = cry[lane];
                uint32_t n = cc;
#pragma unroll
                for (int blk = 0; blk < WP_BLK; ++blk) {
                    const uint32_t m = masks[wp_swz(b, blk)];
                    if ((m >> lane) & 1u) stg[off + n + (uint32_t)__popc(m & lt)] = vb + 32u * (uint32_t)blk;
                    n += (uint32_t)__popc(m);
                }
                // write [0, end): everything on the last tile, else up to the
                // last sector boundary of the run
                const uint64_t ea = (o + n) & ~7ull;
                const uint32_t end = last ? n : (ea > o ? (uint32_t)(ea - o) : 0u);
                __syncwarp();
                if ((uint32_t)lane < n - end) cry[lane] = stg[off + end + lane];
                if (lane == (b & 31)) {                       // running position / carry of source b
                    if (b < 32) { o_lo += end; cc_lo = n - end; }
                    else { o_hi += end; cc_hi = n - end; }
                }
                if (end == 0) continue;
                const uint32_t sid = __shfl_sync(0xffffffffu, b < 32 ? sid_lo : sid_hi, b & 31);
                uint32_t *dp = odst + o, *sp = osrc + o;
                if (!vec_ok) {
                    for (uint32_t e = (uint32_t)lane; e < end; e += 32) { dp[e] = stg[off + e]; sp[e] = sid; }
                    continue;
                }
                const uint32_t h = min(end, (4u - off) & 3u);              // head up to 16-B alignment
                const uint32_t nv = (end - h) >> 2;                         // 16-B vectors
                const uint32_t t0 = h + 4u * nv;                            // tail (< 4 elements)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    if (nv) bulk_s2g(dp + h, stg + off + h, nv * 16u);
                    bulk_commit();
                }
                sbuf ^= 1;
                if ((uint32_t)lane < h) { dp[lane] = stg[off + lane]; sp[lane] = sid; }
                if (t0 + (uint32_t)lane < end) { dp[t0 + lane] = stg[off + t0 + lane]; sp[t0 + lane] = sid; }
                uint4 *vs = reinterpret_cast<uint4 *>(sp + h);
                const uint4 sv = make_uint4(sid, sid, sid, sid);
                for (uint32_t e = (uint32_t)lane; e < nv; e += 32) vs[e] = sv;
            }
        }
        __syncthreads();                         // every warp is done with the masks
    }
    if (lane == 0) bulk_wait_all();              // bulk stores complete before the CTA exits
}

// epsilon pairs (v, v) of non-productive candidates in [jlo, jhi)
__global__ void k_write_eps(const uint8_t *flag, const uint32_t *cand, uint64_t jlo, uint64_t jhi,
                            const unsigned long long *start, uint32_t *osrc, uint32_t *odst) {
    for (uint64_t j = jlo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < jhi; j += (uint64_t)gridDim.x * blockDim.x) {
        if (flag[j]) continue;
        const unsigned long long o = start[j - jlo];
        osrc[o] = cand[j];
        odst[o] = cand[j];
    }
}

// RPQ_DEBUG_TIMING=1: print host-observed phase times (synchronising);
// RPQ_DEBUG_EVENTS=1: device-side phase times from events (no synchronisation),
// printed when the evaluation ends
struct PhaseTimer {
    bool on, ev;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t;
    std::vector<std::pair<const char *, cudaEvent_t>> evs;
    explicit PhaseTimer(cudaStream_t st)
        : on(getenv("RPQ_DEBUG_TIMING") != nullptr), ev(getenv("RPQ_DEBUG_EVENTS") != nullptr), s(st) {
        t = std::chrono::steady_clock::now();
        mark("begin");
    }
    void mark(const char *what) {
        nvtxMarkA(what);                 // phase boundary on the NVTX timeline
        if (ev) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, s);
            evs.emplace_back(what, e);
        }
        if (!on) return;
        cudaStreamSynchronize(s);
        auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[rpq] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
    ~PhaseTimer() {
        if (!ev) return;
        cudaStreamSynchronize(s);
        for (size_t i = 1; i < evs.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, evs[i - 1].second, evs[i].second);
            fprintf(stderr, "[rpq-ev] %-28s %9.3f ms\n", evs[i].first, ms);
        }
        for (auto &e : evs) cudaEventDestroy(e.second);
    }
};

inline int grid_for(uint64_t threads, int block = 256, int cap = 148 * 16) {
    uint64_t g = (threads + block - 1) / block;
    if (g > (uint64_t)cap) g = cap;
    return g ? (int)g : 1;
}

// Symmetry of one label's edge set: a warp per row u, every neighbour w
// binary-searches u in w's (sorted) row.
__global__ void k_sym_check(const uint32_t *off, const uint32_t *nbr, uint32_t nv, int *bad) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * blockDim.x >> 5;
    for (uint64_t u = wid; u < nv; u += nwarps) {
        if (*(volatile int *)bad) return;
        const uint32_t b = off[u], e = off[u + 1];
        bool ok = true;
        for (uint32_t j = b + lane; j < e; j += 32) {
            const uint32_t w = nbr[j];
            uint32_t lo = off[w], hi = off[w + 1];
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (nbr[mid] < (uint32_t)u) lo = mid + 1; else hi = mid;
            }
            ok &= lo < off[w + 1] && nbr[lo] == (uint32_t)u;
        }
        if (!__all_sync(0xffffffffu, ok)) {
            if (lane == 0) atomicExch(bad, 1);
            return;
        }
    }
}

// Cached per graph and label (first use only; not query work after that).
bool label_symmetric(const rpq_graph *g, uint32_t l, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g->sym_mu);
    if (g->sym.size() != g->csr.size()) g->sym.assign(g->csr.size(), -1);
    if (g->sym[l] >= 0) return g->sym[l] != 0;
    int *d_bad = (int *)dev_alloc(sizeof(int), s);
    int bad = 1;
    if (d_bad && cudaMemsetAsync(d_bad, 0, sizeof(int), s) == cudaSuccess) {
        k_sym_check<<<148 * 8, 256, 0, s>>>(g->csr[l].off, g->csr[l].nbr, g->nv, d_bad);
        if (cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            bad = 1;
    }
    cudaGetLastError();
    dev_free(d_bad, s);
    g->sym[l] = bad ? 0 : 1;
    return !bad;
}

// ---- host-side evaluation driver ------------------------------------------
struct Workspace {
    cudaStream_t s;
    std::vector<void *> ptrs;
    ~Workspace() { for (void *p : ptrs) dev_free(p, s); }
    void *get(size_t bytes) {
        void *p = dev_alloc(bytes, s);
        if (p) ptrs.push_back(p);
        return p;
    }
};

struct Range { uint32_t lo, hi; bool empty() const { return lo > hi; } };

Range hull(Range a, Range b) {
    if (a.empty()) return b;
    if (b.empty()) return a;
    return {std::min(a.lo, b.lo), std::max(a.hi, b.hi)};
}

// Level loop, device-driven: a CUDA graph whose body is a conditional WHILE
// node running two levels (parity 0, then 1) per iteration; the end kernel
// sets the loop condition from the "activated" flag, so a whole batch runs
// without a host round trip per level.  (An empty extra level costs one
// scan of the tiny XB bitmap.)
struct LevelGraph {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle h{};
    std::vector<cudaGraphNode_t> nodes;   // body kernel nodes, in build order
    ~LevelGraph() {
        if (exec) cudaGraphExecDestroy(exec);
        if (g) cudaGraphDestroy(g);
    }
};

// update = true: LG holds an instantiated graph of the same topology (same
// kernels and node order); only the kernel arguments and grids are patched
// into its body nodes (cudaGraphExecKernelNodeSetParams, microseconds)
// instead of a new instantiation (~0.3 ms on a cold query, e.g. a new graph).
template <bool STATS, bool BND>
cudaError_t build_level_graph(LevelGraph &LG, const DevAuto &A, const Layout *Sg, const LevelArgs &P0,
                              const LevelArgs &P1, int grid, int hgrid, uint64_t nxbwords, bool hub,
                              bool update = false) {
    cudaError_t e;
    cudaGraph_t body = nullptr;
    if (!update) {
        if ((e = cudaGraphCreate(&LG.g, 0)) != cudaSuccess) return e;
        if ((e = cudaGraphConditionalHandleCreate(&LG.h, LG.g, 1, cudaGraphCondAssignDefault)) != cudaSuccess) return e;
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = LG.h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cn;
        if ((e = cudaGraphAddNode(&cn, LG.g, nullptr, 0, &cp)) != cudaSuccess) return e;
        body = cp.conditional.phGraph_out[0];
        LG.nodes.clear();
    }
    cudaGraphNode_t prev = nullptr;
    size_t ni = 0;
    auto add = [&](void *fn, dim3 gr, dim3 bl, void **args, unsigned smem = 0) -> cudaError_t {
        cudaKernelNodeParams kp{};
        kp.func = fn;
        kp.gridDim = gr;
        kp.blockDim = bl;
        kp.sharedMemBytes = smem;
        kp.kernelParams = args;
        if (update) {
            if (ni >= LG.nodes.size()) return cudaErrorInvalidValue;
            return cudaGraphExecKernelNodeSetParams(LG.exec, LG.nodes[ni++], &kp);
        }
        cudaGraphNode_t n;
        cudaError_t r = cudaGraphAddKernelNode(&n, body, prev ? &prev : nullptr, prev ? 1 : 0, &kp);
        prev = n;
        LG.nodes.push_back(n);
        return r;
    };
    cudaGraphConditionalHandle h = LG.h;
    DevAuto a = A;
    const Layout *sg = Sg;
    LevelArgs p0 = P0, p1 = P1;
    Ctrl *ctrl = P0.ctrl;
    uint64_t nxb = nxbwords;
    void *a0[] = {&a, &sg, &p0};
    void *a1[] = {&a, &sg, &p1};
    void *r0[] = {&a, &p0};
    void *r1[] = {&a, &p1};
    void *u0[] = {&p0, &nxb};
    void *u1[] = {&p1, &nxb};
    void *m1[] = {&ctrl, &h};
    const int ugrid = (int)std::min<uint64_t>(148 * 4, (nxbwords + 255) / 256 + 1);
    const bool pull = P0.pull_mode != 0;
    if ((e = add((void *)k_units, dim3(ugrid), dim3(256), u0)) != cudaSuccess) return e;
    if (pull && (e = add((void *)k_pull_prep, dim3(148 * 8), dim3(256), r0)) != cudaSuccess) return e;
    void *lvl = (P0.tma & 1u) ? (void *)k_level<STATS, false, true> : (void *)k_level<STATS, BND>;
    const int lgr = (P0.tma & 1u) ? 148 * RPQ_TMA_MINB : grid;
    const unsigned lsm = (P0.tma & 1u) ? TMA_SMEM : 0u;
    if ((e = add(lvl, dim3(lgr), dim3(256), a0, lsm)) != cudaSuccess) return e;
    if (pull && (e = add((void *)k_pull<STATS>, dim3(148 * 8), dim3(256), a0)) != cudaSuccess) return e;
    void *hubk = (P0.tma & 2u) ? (void *)k_level_hub<STATS, false, true> : (void *)k_level_hub<STATS, BND>;
    const int hgr = (P0.tma & 2u) ? 148 * RPQ_TMA_MINB : hgrid;
    const unsigned hsm = (P0.tma & 2u) ? TMA_SMEM : 0u;
    if (hub && (e = add(hubk, dim3(hgr), dim3(256), a0, hsm)) != cudaSuccess) return e;
    if ((e = add((void *)k_units, dim3(ugrid), dim3(256), u1)) != cudaSuccess) return e;
    if (pull && (e = add((void *)k_pull_prep, dim3(148 * 8), dim3(256), r1)) != cudaSuccess) return e;
    if ((e = add(lvl, dim3(lgr), dim3(256), a1, lsm)) != cudaSuccess) return e;
    if (pull && (e = add((void *)k_pull<STATS>, dim3(148 * 8), dim3(256), a1)) != cudaSuccess) return e;
    if (hub && (e = add(hubk, dim3(hgr), dim3(256), a1, hsm)) != cudaSuccess) return e;
    if ((e = add((void *)k_level_end, dim3(1), dim3(1), m1)) != cudaSuccess) return e;
    if (update) return ni == LG.nodes.size() ? cudaSuccess : cudaErrorInvalidValue;
    return cudaGraphInstantiate(&LG.exec, LG.g, 0);
}

// Level loop, host-driven (RPQ_HOST_LOOP=1, or if graph creation fails):
// one flag readback per level.
rpq_status run_levels_host(const DevAuto &A, const Layout *Sg, const LevelArgs &P0, const LevelArgs &P1, int grid,
                           int hgrid, uint64_t nxbwords, cudaStream_t s, bool stats, uint32_t *h_flag,
                           rpq_stats *out_stats, bool hub) {
    int par = 0;
    const int ugrid = (int)std::min<uint64_t>(148 * 4, (nxbwords + 255) / 256 + 1);
    for (;;) {
        const LevelArgs &P = par ? P1 : P0;
        k_units<<<ugrid, 256, 0, s>>>(P, nxbwords);
        if (P.pull_mode) k_pull_prep<<<148 * 8, 256, 0, s>>>(A, P);
        if (stats) {
            if (P.bounded) k_level<true, true><<<grid, 256, 0, s>>>(A, Sg, P);
            else if (P.tma & 1u) k_level<true, false, true><<<148 * RPQ_TMA_MINB, 256, TMA_SMEM, s>>>(A, Sg, P);
            else k_level<true><<<grid, 256, 0, s>>>(A, Sg, P);
            if (P.pull_mode) k_pull<true><<<148 * 8, 256, 0, s>>>(A, Sg, P);
            if (hub && P.bounded) k_level_hub<true, true><<<hgrid, 256, 0, s>>>(A, Sg, P);
            else if (hub && (P.tma & 2u)) k_level_hub<true, false, true><<<148 * RPQ_TMA_MINB, 256, TMA_SMEM, s>>>(A, Sg, P);
            else if (hub) k_level_hub<true><<<hgrid, 256, 0, s>>>(A, Sg, P);
        } else {
            if (P.bounded) k_level<false, true><<<grid, 256, 0, s>>>(A, Sg, P);
            else if (P.tma & 1u) k_level<false, false, true><<<148 * RPQ_TMA_MINB, 256, TMA_SMEM, s>>>(A, Sg, P);
            else k_level<false><<<grid, 256, 0, s>>>(A, Sg, P);
            if (P.pull_mode) k_pull<false><<<148 * 8, 256, 0, s>>>(A, Sg, P);
            if (hub && P.bounded) k_level_hub<false, true><<<hgrid, 256, 0, s>>>(A, Sg, P);
            else if (hub && (P.tma & 2u)) k_level_hub<false, false, true><<<148 * RPQ_TMA_MINB, 256, TMA_SMEM, s>>>(A, Sg, P);
            else if (hub) k_level_hub<false><<<hgrid, 256, 0, s>>>(A, Sg, P);
        }
        RPQ_CUDA_TRY(cudaMemcpyAsync(h_flag, &P.ctrl->active[par ^ 1], 4, cudaMemcpyDeviceToHost, s));
        RPQ_CUDA_TRY(cudaStreamSynchronize(s));
        RPQ_CUDA_TRY(cudaGetLastError());
        out_stats->kernel_launches += 3;
        par ^= 1;
        if (*h_flag == 0) break;
    }
    return RPQ_OK;
}

}  // namespace

// Evaluate the RPQ from the sorted, distinct candidate sources cand[0..nsrc)
// (device array).  cand == nullptr means all of V (all-pairs, reading R11).
static rpq_status eval_sources_impl(const rpq_graph *g, const rpq_nfa *a, const uint32_t *d_cand_in, uint64_t nsrc,
                                    const rpq_eval_opts *opts_in, rpq_result **out, bool *budget_cached) {
    rpq_eval_opts o{};
    if (opts_in) o = *opts_in;
    if (o.mode == 0) o.mode = RPQ_COUNT;
    const bool want_pairs = o.mode & RPQ_PAIRS;
    const bool want_ps = (o.mode & RPQ_PER_SOURCE) || want_pairs;
    const bool stats = o.mode & RPQ_STATS;
    // PE (product edges traversed, reading R12) from the post-pass only, no
    // in-kernel counters: fused into the COUNT pass (dense and touched paths)
    const bool want_pe = stats || (o.mode & RPQ_PE);
    // length-bounded RPQ ("enforced by controlling traversal
    // depth"): only paths of <= max_hops edges; exact BFS levels (reading D3)
    const bool bounded = (o.mode & RPQ_BOUNDED) != 0;
    const uint32_t max_hops = o.max_hops;
    const bool timeit = o.mode & RPQ_TIME_KERNELS;
    const uint32_t shard_count = o.shard_count ? o.shard_count : 1;
    if (o.shard_index >= shard_count) return rpq_fail(RPQ_EINVAL, "shard_index >= shard_count");
    // the automaton's vocabulary must be the graph's, or a prefix of it
    // (labels added since with rpq_graph_add_label keep the old ids)
    if (a->vocab.size() > g->label_names.size() ||
        !std::equal(a->vocab.begin(), a->vocab.end(), g->label_names.begin()))
        return rpq_fail(RPQ_EINVAL, "automaton was compiled against a different label vocabulary");
    RPQ_CUDA_TRY(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)o.cuda_stream;
    Workspace ws{s, {}};

    rpq_result *res = new rpq_result();
    res->stream = (void *)s;
    res->alloc_snap = alloc_snapshot();
    res->device = g->device;
    auto fail = [&](rpq_status st) { rpq_result_release(res); return st; };
    cudaEvent_t evt0, evt1, e_begin, e_end;
    cudaEventCreate(&evt0); cudaEventCreate(&evt1); cudaEventCreate(&e_begin); cudaEventCreate(&e_end);
    struct EvGuard { cudaEvent_t *e; ~EvGuard() { for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]); } };
    cudaEvent_t evs[4] = {evt0, evt1, e_begin, e_end};
    EvGuard eg{evs};
    cudaEventRecord(e_begin, s);
    PhaseTimer PT(s);
    // RPQ_DEBUG_HOST=1: report host calls of the driver that take > 1 ms
    const bool dbg_host = getenv("RPQ_DEBUG_HOST") != nullptr;
    auto h_t = std::chrono::steady_clock::now();
    auto HM = [&](const char *what) {
        if (!dbg_host) return;
        auto n = std::chrono::steady_clock::now();
        double ms = std::chrono::duration<double, std::milli>(n - h_t).count();
        if (ms > 1.0) fprintf(stderr, "[rpq-host] %-28s %9.3f ms\n", what, ms);
        h_t = n;
    };
    rpq_stats &ST = res->stats;

    // ---- device automaton ------------------------------------------------
    DevAuto A{};
    A.nq = a->nq;
    A.final_mask = a->final_mask;
    std::vector<uint32_t> slot_label;
    for (uint32_t q = 0; q <= a->nq; ++q) A.toff[q] = (uint16_t)a->off[q];
    for (size_t t = 0; t < a->from.size(); ++t) {
        uint32_t l = a->label[t];
        auto it = std::find(slot_label.begin(), slot_label.end(), l);
        int slot = (int)(it - slot_label.begin());
        if (it == slot_label.end()) slot_label.push_back(l);
        A.tslot[t] = (uint8_t)slot;
        A.tto[t] = (uint8_t)a->to[t];
    }
    // reserved bit 1 (rpq_eval_targets): traverse the in-edge CSR, i.e. the
    // transposed graph, with the reversed automaton
    const bool reverse = (o.reserved & 2u) != 0;
    if (reverse && g->in_csr.size() != g->csr.size())
        return fail(rpq_fail(RPQ_EUNSUPPORTED, "graph loaded without RPQ_GRAPH_IN_EDGES"));
    const std::vector<LabelCSR> &CSR = reverse ? g->in_csr : g->csr;
    // Bottom-up (pull) levels need each label's transposed CSR.  Default:
    // only when every label of the query is symmetric (undirected relations
    // such as knows: BFS rows then fill from their first in-neighbours, and
    // the transposed CSR is the CSR itself); RPQ_PULL=always also uses the
    // in-edge CSR of directed labels; RPQ_PULL=never disables it.  (On the
    // directed cfg2 / RMAT queries bottom-up levels measured 1.3-2x slower
    // than top-down ones at every frontier density.)
    const std::vector<LabelCSR> &TCSR = reverse ? g->csr : g->in_csr;
    const bool have_t = TCSR.size() == CSR.size();
    int pull_req = 1;
    {
        const char *pm = getenv("RPQ_PULL");
        if (pm && (!strcmp(pm, "0") || !strcmp(pm, "never"))) pull_req = 0;
        if (pm && (!strcmp(pm, "2") || !strcmp(pm, "always"))) pull_req = 2;
    }
    bool all_sym = pull_req != 0 && !slot_label.empty();
    for (size_t k = 0; k < slot_label.size() && all_sym; ++k) all_sym = label_symmetric(g, slot_label[k], s);
    const bool use_t = pull_req == 2 && have_t && !all_sym;
    for (size_t k = 0; k < slot_label.size(); ++k) {
        A.off[k] = CSR[slot_label[k]].off;
        A.nbr[k] = CSR[slot_label[k]].nbr;
        A.ioff[k] = use_t ? TCSR[slot_label[k]].off : all_sym ? A.off[k] : nullptr;
        A.inbr[k] = use_t ? TCSR[slot_label[k]].nbr : all_sym ? A.nbr[k] : nullptr;
    }
    const bool pull_avail = all_sym || use_t;
    // the hub kernel only runs if some label of the query has rows longer
    // than HUB_EDGES (RMAT); otherwise its launches are left out of the loop
    bool need_hub = getenv("RPQ_ALWAYS_HUB") != nullptr;
    for (size_t k = 0; k < slot_label.size(); ++k) need_hub |= CSR[slot_label[k]].max_deg > HUB_EDGES;
    {   // transitions grouped by target state
        uint32_t k = 0;
        for (uint32_t q2 = 0; q2 < a->nq; ++q2) {
            A.itoff[q2] = (uint16_t)k;
            for (size_t t = 0; t < a->from.size(); ++t)
                if (a->to[t] == q2) { A.itfrom[k] = (uint8_t)a->from[t]; A.itslot[k] = A.tslot[t]; ++k; }
        }
        A.itoff[a->nq] = (uint16_t)k;
    }

    // ---- candidate sources and the productive subset P --------------------
    // all-pairs: the candidates 0..|V|-1 and the productive set come from
    // the graph's plan cache (no device round trip after the first query)
    const bool allpairs = d_cand_in == nullptr;
    const uint32_t *cand = d_cand_in;
    std::unique_lock<std::mutex> plan_lk(g->plan_mu, std::defer_lock);
    if (!cand) {
        nsrc = g->nv;
        plan_lk.lock();
        if (!g->d_iota) {
            uint32_t *iota = (uint32_t *)graph_alloc(g, nsrc * 4, s);
            if (!iota) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (sources)"));
            k_iota<<<grid_for(nsrc), 256, 0, s>>>(iota, nsrc);
            ST.kernel_launches++;
            g->d_iota = iota;
        }
        cand = g->d_iota;
        plan_lk.unlock();
    }
    // q0's labels (plan-cache key of the productive set)
    std::vector<uint32_t> q0_labels;
    for (uint32_t t = a->nq ? a->off[0] : 0; a->nq && t < a->off[1]; ++t) q0_labels.push_back(a->label[t]);
    std::sort(q0_labels.begin(), q0_labels.end());
    q0_labels.erase(std::unique(q0_labels.begin(), q0_labels.end()), q0_labels.end());
    uint8_t *flag = (uint8_t *)ws.get(std::max<uint64_t>(nsrc, 1));
    uint32_t *pidx = nullptr;
    const std::vector<uint32_t> *h_pidx = nullptr;   // host copy (all-pairs, cached)
    uint64_t *d_np = (uint64_t *)ws.get(32);
    if (!flag || !d_np) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (sources)"));
    uint64_t np = 0;
    uint32_t p_first_d = 0, p_last_d = 0;
    if (nsrc && a->nq) {
        k_productive<<<grid_for(nsrc), 256, 0, s>>>(A, cand, nsrc, flag);
        ST.kernel_launches++;
    }
    if (allpairs && nsrc && a->nq) {
        std::lock_guard<std::mutex> lk(g->plan_mu);
        for (auto *e : g->prod_cache)
            if (e->reverse == (reverse ? 1u : 0u) && e->labels == q0_labels) {
                pidx = e->d_pidx;
                h_pidx = &e->h_pidx;
            }
    }
    if (h_pidx) {
        np = h_pidx->size();
        p_first_d = np ? (*h_pidx)[0] : 0;            // cand = iota: vertex id = index
        p_last_d = np ? (*h_pidx)[np - 1] : 0;
    } else if (nsrc && a->nq) {
        pidx = (uint32_t *)ws.get(std::max<uint64_t>(nsrc, 1) * 4);
        if (!pidx) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (sources)"));
        size_t tb = 0;
        thrust::counting_iterator<uint32_t> it(0);
        cub::DeviceSelect::Flagged(nullptr, tb, it, flag, pidx, d_np, (int64_t)nsrc, s);
        void *tmp = ws.get(tb);
        if (!tmp) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory"));
        cub::DeviceSelect::Flagged(tmp, tb, it, flag, pidx, d_np, (int64_t)nsrc, s);
        // |P| and the first / last productive source in one readback
        k_prod_bounds<<<1, 32, 0, s>>>(d_np, pidx, cand, d_np + 1);
        uint64_t hb3[3] = {0, 0, 0};
        RPQ_CUDA_TRY(cudaMemcpyAsync(hb3, d_np + 1, 24, cudaMemcpyDeviceToHost, s));
        RPQ_CUDA_TRY(cudaStreamSynchronize(s));
        np = hb3[0];
        p_first_d = (uint32_t)hb3[1];
        p_last_d = (uint32_t)hb3[2];
        HM("np readback");
        if (allpairs) {   // remember the productive set for the next query on this graph
            auto *e = new rpq_graph::ProdEntry();
            e->reverse = reverse ? 1u : 0u;
            e->labels = q0_labels;
            e->h_pidx.resize(np);
            e->d_pidx = (uint32_t *)graph_alloc(g, std::max<uint64_t>(np, 1) * 4, s);
            if (!e->d_pidx) {
                delete e;
            } else {
                if (np) {
                    RPQ_CUDA_TRY(cudaMemcpyAsync(e->d_pidx, pidx, np * 4, cudaMemcpyDeviceToDevice, s));
                    RPQ_CUDA_TRY(cudaMemcpyAsync(e->h_pidx.data(), pidx, np * 4, cudaMemcpyDeviceToHost, s));
                    RPQ_CUDA_TRY(cudaStreamSynchronize(s));
                }
                std::lock_guard<std::mutex> lk(g->plan_mu);
                g->prod_cache.push_back(e);
                h_pidx = &e->h_pidx;
            }
        }
    } else if (nsrc) {
        RPQ_CUDA_TRY(cudaMemsetAsync(flag, 0, nsrc, s));
    }
    if (!pidx) {
        pidx = (uint32_t *)ws.get(std::max<uint64_t>(nsrc, 1) * 4);
        if (!pidx) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (sources)"));
    }
    ST.productive_sources = np;
    PT.mark("productive sources");
    const bool eps = a->accepts_empty;

    // ---- ranges per state (hull of dst ranges of entering labels) ---------
    std::vector<Range> in_range(a->nq, Range{1, 0});
    for (size_t t = 0; t < a->from.size(); ++t) {
        const LabelCSR &c = CSR[a->label[t]];
        in_range[a->to[t]] = hull(in_range[a->to[t]], Range{c.dst_min, c.dst_max});
    }

    // q0 needs rows only if something can enter it or it is final (its row
    // then carries the epsilon pair); otherwise level 0 expands the seeds
    // directly (k_seed_expand)
    bool q0_entered = false;
    for (size_t t = 0; t < a->to.size(); ++t) q0_entered |= a->to[t] == 0;
    const bool skip_q0 = a->nq > 0 && !q0_entered && !((a->final_mask >> 0) & 1ull) && !getenv("RPQ_NO_SKIP_Q0");
    // a final state without outgoing transitions collects result bits
    // without activity bitmaps, so its rows are not in the touched sets:
    // such automata clear and count densely
    int dead_final = bounded ? 1 : 0;   // (bounded: the last level's bits are in no touched set)
    for (uint32_t q = 0; q < a->nq; ++q)
        if (((a->final_mask >> q) & 1ull) && a->off[q + 1] == a->off[q]) dead_final = 1;

    // ---- batch plan -------------------------------------------------------
    // Rows of the worst batch (q0 range = hull of all productive sources) set
    // the word budget: 3 state arrays x 8 B + worklists/bitmaps per word.
    const uint32_t p_first = p_first_d, p_last = p_last_d;
    HM("p_first/p_last");
    uint64_t R_max = 0;
    for (uint32_t q = 0; q < a->nq; ++q) {
        Range r = in_range[q];
        if (q == 0 && np && !skip_q0) r = hull(r, Range{p_first, p_last});
        R_max += r.empty() ? 0 : (uint64_t)r.hi - r.lo + 1;
    }
    // global row indices (state, vertex) are u32 inside the level kernels
    if (R_max >= (1ull << 32))
        return fail(rpq_fail(RPQ_EUNSUPPORTED, "%llu state rows (sum of per-state vertex ranges) >= 2^32",
                             (unsigned long long)R_max));
    // Sharded evaluations must cut the sources into the SAME batches on every
    // rank (batch b -> shard b % shard_count): the automatic width depends on
    // this device's free memory, so it is only allowed with an explicit
    // budget; rpq_plan + an all-reduce MIN (rpq_eval_allpairs_dist in the
    // Python layer) agrees on one width.
    if (shard_count > 1 && o.batch_sources == 0 && o.hbm_budget_bytes == 0 && !(o.reserved & 4u))
        return fail(rpq_fail(RPQ_EINVAL, "shard_count > 1 needs batch_sources or hbm_budget_bytes (ranks must agree "
                                         "on the batch plan; see rpq_plan)"));
    uint64_t budget = o.hbm_budget_bytes ? o.hbm_budget_bytes : (uint64_t)(dev_available(budget_cached) * 0.9);
    HM("dev_available");
    uint64_t B = o.batch_sources;
    if (B == 0) {
        // bytes per 64-source word column: Vis + Done, bitmaps, and for
        // PER_SOURCE / PAIRS the per-(source, 1024-vertex tile) counts; the
        // materialised pairs are allocated outside the budget, so those modes
        // keep half of it free
        double per_word = (bounded ? 24.0 : 16.0) * R_max + 0.5 * R_max + 64.0 * 8 * 2;
        uint64_t bud = budget;
        if (want_ps) {
            uint64_t hullv = 0;
            for (uint32_t q = 0; q < a->nq; ++q)
                if ((a->final_mask >> q) & 1) {
                    Range r = in_range[q];
                    if (q == 0 && np) r = hull(r, Range{p_first, p_last});
                    hullv = std::max<uint64_t>(hullv, r.empty() ? 0 : (uint64_t)r.hi - r.lo + 1);
                }
            per_word += 64.0 * (4.0 * ((double)hullv / TILE_V + 1) + 24.0);
            bud /= 2;
        }
        uint64_t nw_max = per_word > 0 ? (uint64_t)(bud / per_word) : 1;
        if (nw_max < 1) nw_max = 1;
        B = std::min<uint64_t>(std::max<uint64_t>(np, 1), nw_max * 64);
        // Whole row groups: a warp advances and expands KGRP chunks of 32
        // words (2 KB of a row) at a time.  When several batches are needed
        // anyway and the HBM-maximal width leaves the last group of every row
        // mostly empty (RMAT-24: 306 words = 8 + 1.6 chunks), round the width
        // down to whole groups (256 words = 16,384 sources): measured 8 %
        // less time for the same sources on RMAT-24 despite 20 % more batches
        // (scripts/batch_width.py).  A single-batch query keeps its width.
        {
            const uint64_t gw = (uint64_t)KGRP * 32;
            if (B < np && nw_max >= gw && !getenv("RPQ_NO_GROUP_ALIGN")) {
                const double ch = (double)nw_max / 32.0;
                const double groups = std::ceil(ch / KGRP);
                if (ch / (KGRP * groups) < 0.75) B = nw_max / gw * gw * 64;
            }
        }
        // shard-aware: at least one batch per shard, widths in whole words
        if (shard_count > 1) {
            const uint64_t per = ((np + shard_count - 1) / shard_count + 63) / 64 * 64;
            B = std::min<uint64_t>(B, std::max<uint64_t>(per, 64));
        }
    }
    B = std::max<uint64_t>(1, B);
    uint64_t nw = (B + 63) / 64;
    uint32_t CW = o.chunk_words;
    if (CW == 0) { CW = 1; while (CW < 32 && CW < nw) CW <<= 1; }
    if (CW != 1 && CW != 2 && CW != 4 && CW != 8 && CW != 16 && CW != 32)
        return fail(rpq_fail(RPQ_EINVAL, "chunk_words must be 1,2,4,8,16 or 32"));
    nw = (nw + CW - 1) / CW * CW;
    {
        // optional row alignment (RPQ_NW_ALIGN words); measured neutral for
        // cfg2 at 256 words = 2 KB, so off by default
        const char *ea = getenv("RPQ_NW_ALIGN");
        const uint64_t al = ea ? strtoull(ea, nullptr, 10) : 1;
        if (al > 1 && nw >= al) nw = (nw + al - 1) / al * al;
    }
    const uint64_t nchunk = nw / CW;
    const uint64_t nbatches = np ? (np + B - 1) / B : 0;
    ST.batch_sources = (uint32_t)B;
    ST.chunk_words = CW;
    if (o.reserved & 4u) {   // rpq_plan: the batch plan only, nothing evaluated
        ST.batches = (uint32_t)nbatches;
        ST.state_words = R_max * nw;
        *out = res;
        return RPQ_OK;
    }

    // batch boundaries: first/last productive candidate index of each batch
    // and their vertex ids (one kernel + one copy for all batches)
    std::vector<uint32_t> bfirst(nbatches), blast(nbatches), sfirst(nbatches), slast(nbatches);
    if (nbatches && h_pidx) {   // all-pairs: candidate index = vertex id
        for (uint64_t b = 0; b < nbatches; ++b) {
            bfirst[b] = sfirst[b] = (*h_pidx)[b * B];
            blast[b] = slast[b] = (*h_pidx)[std::min<uint64_t>(np, (b + 1) * B) - 1];
        }
    } else if (nbatches) {
        uint32_t *d_bounds = (uint32_t *)ws.get(nbatches * 16);
        if (!d_bounds) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
        k_batch_bounds<<<grid_for(nbatches), 256, 0, s>>>(pidx, cand, np, B, nbatches, d_bounds);
        ST.kernel_launches++;
        std::vector<uint32_t> hb(nbatches * 4);
        RPQ_CUDA_TRY(cudaMemcpyAsync(hb.data(), d_bounds, nbatches * 16, cudaMemcpyDeviceToHost, s));
        RPQ_CUDA_TRY(cudaStreamSynchronize(s));
        for (uint64_t b = 0; b < nbatches; ++b) {
            bfirst[b] = hb[4 * b]; blast[b] = hb[4 * b + 1];
            sfirst[b] = hb[4 * b + 2]; slast[b] = hb[4 * b + 3];
        }
    }
    HM("batch bounds");

    PT.mark("batch plan");
    std::vector<uint64_t> js;   // batch b owns candidates [js[b], js[b+1]) (plan.cpp)
    batch_plan(bfirst.data(), nbatches, nsrc, js);
    auto jstart = [&](uint64_t b) -> uint64_t { return js[b]; };
    const uint64_t nb_eff = std::max<uint64_t>(nbatches, 1);

    // ---- sparse engine: a warp per source when the per-source reach is
    // small (decided on a sample); overflowing sources go to the dense engine
    bool sparse_done = false;
    uint64_t sparse_total = 0, sub_pe = 0;
    rpq_result *sub_keep = nullptr;
    unsigned long long *cand_cnt = nullptr;
    // RPQ_SOURCE_PE: per-candidate product edges (verification mode)
    const bool want_spe = want_ps && (o.mode & RPQ_SOURCE_PE);
    unsigned long long *cand_pe = nullptr, *spe = nullptr;
    if (want_spe) {
        cand_pe = (unsigned long long *)ws.get(std::max<uint64_t>(nsrc, 1) * 8);
        spe = (unsigned long long *)ws.get(std::max<uint64_t>(np, 1) * 8);
        if (!cand_pe || !spe) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (per-source PE)"));
        RPQ_CUDA_TRY(cudaMemsetAsync(cand_pe, 0, std::max<uint64_t>(nsrc, 1) * 8, s));
        RPQ_CUDA_TRY(cudaMemsetAsync(spe, 0, std::max<uint64_t>(np, 1) * 8, s));
    }
    unsigned long long *d_stats = (unsigned long long *)ws.get(NSTAT * 8 + 8);
    if (!d_stats) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
    unsigned long long *d_total = d_stats + NSTAT;
    RPQ_CUDA_TRY(cudaMemsetAsync(d_stats, 0, NSTAT * 8 + 8, s));
    {
        const char *eng = getenv("RPQ_ENGINE");
        const bool force_dense = (o.reserved & 1u) || bounded || (eng && !strcmp(eng, "dense"));
        const bool force_sparse = eng && !strcmp(eng, "sparse");
        if (np && !force_dense) {
            unsigned long long *sc = (unsigned long long *)ws.get(np * 8);
            uint8_t *sov = (uint8_t *)ws.get(np);            // warp tier overflowed -> dense engine
            uint8_t *tov = (uint8_t *)ws.get(np);            // thread tier overflowed -> warp tier
            uint32_t *tlist = (uint32_t *)ws.get(np * 4);    // ... their productive indices
            uint64_t *d_nt = (uint64_t *)ws.get(8);
            if (!sc || !sov || !tov || !tlist || !d_nt)
                return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (sparse)"));
            bool use = force_sparse;
            // all-pairs: the engine decision is a property of (graph,
            // automaton) -- cached in the graph after the first sample
            std::vector<uint32_t> sig;
            int cached = -1;
            if (allpairs && !use) {
                sig = {reverse ? 1u : 0u, a->nq, (uint32_t)a->final_mask, (uint32_t)(a->final_mask >> 32)};
                for (size_t t = 0; t < a->from.size(); ++t) {
                    sig.push_back(a->from[t]);
                    sig.push_back(a->label[t]);
                    sig.push_back(a->to[t]);
                }
                std::lock_guard<std::mutex> lk(g->plan_mu);
                for (auto &e : g->engine_cache)
                    if (e.first == sig) cached = e.second;
            }
            if (cached >= 0) use = cached != 0;
            if (!use && cached < 0) {
                // two stages: 256 evenly spread sources settle clearly dense
                // queries (>= 25 % overflow; the warp tier's 1,024-key probe
                // of 2,048 sources cost ~0.3 ms per cold query), otherwise
                // 2,048 sources decide (<= 2 % overflow -> sparse engine)
                unsigned long long *d_nov = (unsigned long long *)ws.get(8);
                if (!d_nov) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                const uint64_t stage_ns[2] = {std::min<uint64_t>(np, 256), std::min<uint64_t>(np, 2048)};
                for (int stage = 0; stage < 2; ++stage) {
                    const uint64_t ns = stage_ns[stage];
                    uint32_t *didx = (uint32_t *)ws.get(ns * 4);
                    if (!didx) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                    k_sample_idx<<<grid_for(ns), 256, 0, s>>>(didx, ns, np);   // k * np / ns, evenly spread
                    k_sparse<false, false><<<grid_for(ns * 32, SP_WARPS * 32, 148 * 8), SP_WARPS * 32, 0, s>>>(
                        A, cand, pidx, didx, ns, B, 0, 1, sc, sov, d_stats);
                    // overflow flags of the sampled indices, summed on the device
                    k_sum_flags<<<1, 256, 0, s>>>(sov, didx, ns, d_nov);
                    ST.kernel_launches += 3;
                    unsigned long long nov = 0;
                    RPQ_CUDA_TRY(cudaMemcpyAsync(&nov, d_nov, 8, cudaMemcpyDeviceToHost, s));
                    RPQ_CUDA_TRY(cudaStreamSynchronize(s));
                    HM("sparse sample");
                    use = nov * 50 <= ns;
                    if (stage == 0 && (nov * 4 >= ns || ns == stage_ns[1])) break;
                }
                if (allpairs) {
                    std::lock_guard<std::mutex> lk(g->plan_mu);
                    g->engine_cache.emplace_back(sig, use ? 1 : 0);
                }
            }
            if (use) {
                // full pass over this shard's productive sources
                RPQ_CUDA_TRY(cudaMemsetAsync(sc, 0, np * 8, s));
                RPQ_CUDA_TRY(cudaMemsetAsync(sov, 0, np, s));
                cudaEvent_t sp0 = nullptr, sp1 = nullptr;
                if (timeit) { cudaEventCreate(&sp0); cudaEventCreate(&sp1); cudaEventRecord(sp0, s); }
                // thread tier over every source of the shard, then the warp
                // tier over the sources the thread tier could not hold
                RPQ_CUDA_TRY(cudaMemsetAsync(tov, 0, np, s));
                if (want_pe)
                    k_sparse_thread<true, false><<<grid_for(np), 256, 0, s>>>(A, cand, pidx, np, B, o.shard_index,
                                                                             shard_count, sc, tov, d_stats, nullptr,
                                                                             nullptr, nullptr, spe);
                else
                    k_sparse_thread<false, false><<<grid_for(np), 256, 0, s>>>(A, cand, pidx, np, B, o.shard_index,
                                                                              shard_count, sc, tov, d_stats, nullptr,
                                                                              nullptr, nullptr, spe);
                {
                    size_t tt = 0;
                    thrust::counting_iterator<uint32_t> itt(0);
                    cub::DeviceSelect::Flagged(nullptr, tt, itt, tov, tlist, d_nt, (int64_t)np, s);
                    void *tmpt = ws.get(tt);
                    if (!tmpt) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                    cub::DeviceSelect::Flagged(tmpt, tt, itt, tov, tlist, d_nt, (int64_t)np, s);
                }
                if (want_pe)
                    k_sparse<true, false><<<148 * 8, SP_WARPS * 32, 0, s>>>(A, cand, pidx, tlist, np, B, o.shard_index,
                                                                     shard_count, sc, sov, d_stats, nullptr, nullptr,
                                                                     nullptr, nullptr, d_nt, spe);
                else
                    k_sparse<false, false><<<148 * 8, SP_WARPS * 32, 0, s>>>(A, cand, pidx, tlist, np, B, o.shard_index,
                                                                      shard_count, sc, sov, d_stats, nullptr, nullptr,
                                                                      nullptr, nullptr, d_nt, spe);
                ST.kernel_launches += 3;
                if (timeit) {
                    cudaEventRecord(sp1, s);
                    cudaEventSynchronize(sp1);
                    float ms = 0;
                    cudaEventElapsedTime(&ms, sp0, sp1);
                    ST.expand_ms += ms;
                    cudaEventDestroy(sp0);
                    cudaEventDestroy(sp1);
                }
                ST.expand_launches += 1;
                // overflowed sources -> dense sub-evaluation
                uint32_t *olist = (uint32_t *)ws.get(np * 4);
                uint64_t *d_no = (uint64_t *)ws.get(8);
                unsigned long long *d_sum = (unsigned long long *)ws.get(8);
                if (!olist || !d_no || !d_sum) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                size_t t1 = 0, t2 = 0;
                thrust::counting_iterator<uint32_t> itc(0);
                cub::DeviceSelect::Flagged(nullptr, t1, itc, sov, olist, d_no, (int64_t)np, s);
                cub::DeviceReduce::Sum(nullptr, t2, sc, d_sum, (int64_t)np, s);
                void *tmp = ws.get(std::max(t1, t2));
                if (!tmp) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                cub::DeviceSelect::Flagged(tmp, t1, itc, sov, olist, d_no, (int64_t)np, s);
                cub::DeviceReduce::Sum(tmp, t2, sc, d_sum, (int64_t)np, s);
                uint64_t no = 0;
                unsigned long long ssum = 0;
                RPQ_CUDA_TRY(cudaMemcpyAsync(&no, d_no, 8, cudaMemcpyDeviceToHost, s));
                RPQ_CUDA_TRY(cudaMemcpyAsync(&ssum, d_sum, 8, cudaMemcpyDeviceToHost, s));
                RPQ_CUDA_TRY(cudaStreamSynchronize(s));
                sparse_total = ssum;
                // epsilon pairs of the non-productive candidates in this shard's batches
                if (eps)
                    for (uint64_t b = o.shard_index; b < nb_eff; b += shard_count) {
                        const uint64_t nbp = b < nbatches ? std::min<uint64_t>(B, np - b * B) : 0;
                        sparse_total += (js[b + 1] - js[b]) - nbp;
                    }
                if (want_ps) {
                    cand_cnt = (unsigned long long *)ws.get(std::max<uint64_t>(nsrc, 1) * 8);
                    if (!cand_cnt) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (counts)"));
                    k_fill_eps<<<grid_for(nsrc), 256, 0, s>>>(cand_cnt, nsrc, eps ? 1ull : 0ull);
                    k_sparse_scatter<<<grid_for(np), 256, 0, s>>>(pidx, sc, sov, np, B, o.shard_index, shard_count,
                                                                 cand_cnt);
                    if (want_spe)
                        k_sparse_scatter<<<grid_for(np), 256, 0, s>>>(pidx, spe, sov, np, B, o.shard_index,
                                                                     shard_count, cand_pe);
                    ST.kernel_launches += 2;
                }
                if (no) {
                    uint32_t *osrc = (uint32_t *)ws.get(no * 4);
                    if (!osrc) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                    k_gather_idx<<<grid_for(no), 256, 0, s>>>(cand, pidx, olist, no, osrc);
                    ST.kernel_launches++;
                    rpq_eval_opts so = o;
                    so.reserved |= 1u;               // dense only
                    so.shard_index = 0;
                    so.shard_count = 1;
                    so.mode = (o.mode & (RPQ_STATS | RPQ_TIME_KERNELS | RPQ_PE | RPQ_SOURCE_PE)) |
                              (want_pairs ? RPQ_PAIRS : want_ps ? RPQ_PER_SOURCE : RPQ_COUNT);
                    rpq_result *sub = nullptr;
                    rpq_status sst = eval_sources_device(g, a, osrc, no, &so, &sub);
                    if (sst != RPQ_OK) return fail(sst);
                    struct SubGuard { rpq_result *r; ~SubGuard() { rpq_result_release(r); } } sg{sub};
                    sparse_total += sub->count;
                    const rpq_stats &ss = sub->stats;
                    ST.word_items += ss.word_items; ST.word_edge_ops += ss.word_edge_ops; ST.items += ss.items;
                    ST.item_edges += ss.item_edges; ST.item_transitions += ss.item_transitions;
                    ST.activations += ss.activations; ST.next_reds += ss.next_reds; ST.levels += ss.levels;
                    ST.batches += ss.batches; ST.expand_launches += ss.expand_launches;
                    ST.kernel_launches += ss.kernel_launches; ST.expand_ms += ss.expand_ms;
                    sub_pe = ss.product_edges;
                    if (want_ps && sub->n_ps) {
                        k_scatter_sub<<<grid_for(sub->n_ps), 256, 0, s>>>(
                            cand, nsrc, sub->ps_src, (const unsigned long long *)sub->ps_cnt, sub->n_ps, cand_cnt);
                        if (want_spe && sub->ps_pe)
                            k_scatter_sub<<<grid_for(sub->n_ps), 256, 0, s>>>(
                                cand, nsrc, sub->ps_src, (const unsigned long long *)sub->ps_pe, sub->n_ps, cand_pe);
                        ST.kernel_launches++;
                    }
                    if (want_pairs) {   // keep the sub-result until its pairs are placed
                        sub_keep = sub;
                        sg.r = nullptr;
                    }
                }
                if (want_pairs) {
                    // starts of every candidate (other shards' intervals count 0)
                    for (uint64_t b = 0; b < nb_eff; ++b)
                        if (b % shard_count != o.shard_index && js[b + 1] > js[b])
                            RPQ_CUDA_TRY(cudaMemsetAsync(cand_cnt + js[b], 0, (js[b + 1] - js[b]) * 8, s));
                    unsigned long long *start = (unsigned long long *)ws.get((nsrc + 1) * 8);
                    int *d_err = (int *)ws.get(sizeof(int));
                    if (!start || !d_err) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                    size_t tb = 0;
                    cub::DeviceScan::ExclusiveSum(nullptr, tb, cand_cnt, start, (int64_t)nsrc, s);
                    void *tmp2 = ws.get(tb);
                    if (!tmp2) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                    cub::DeviceScan::ExclusiveSum(tmp2, tb, cand_cnt, start, (int64_t)nsrc, s);
                    unsigned long long ls = 0, lc = 0;
                    RPQ_CUDA_TRY(cudaMemcpyAsync(&ls, start + nsrc - 1, 8, cudaMemcpyDeviceToHost, s));
                    RPQ_CUDA_TRY(cudaMemcpyAsync(&lc, cand_cnt + nsrc - 1, 8, cudaMemcpyDeviceToHost, s));
                    RPQ_CUDA_TRY(cudaMemsetAsync(d_err, 0, sizeof(int), s));
                    RPQ_CUDA_TRY(cudaStreamSynchronize(s));
                    const uint64_t tot = ls + lc;
                    {   // per-batch row ranges of this shard (start = global scan, other shards zeroed)
                        std::vector<uint64_t> bj;
                        for (uint64_t b = o.shard_index; b < nb_eff; b += shard_count) bj.push_back(b);
                        if (!bj.empty()) {
                            std::vector<unsigned long long> hs(bj.size());
                            unsigned long long *d_bs = (unsigned long long *)ws.get(bj.size() * 8);
                            uint64_t *d_bj = (uint64_t *)ws.get(bj.size() * 8);
                            if (!d_bs || !d_bj) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                            for (auto &x : bj) x = js[x];
                            RPQ_CUDA_TRY(cudaMemcpyAsync(d_bj, bj.data(), bj.size() * 8, cudaMemcpyHostToDevice, s));
                            k_gather_u64<<<grid_for(bj.size()), 256, 0, s>>>(start, d_bj, bj.size(), d_bs);
                            RPQ_CUDA_TRY(cudaMemcpyAsync(hs.data(), d_bs, bj.size() * 8, cudaMemcpyDeviceToHost, s));
                            RPQ_CUDA_TRY(cudaStreamSynchronize(s));
                            size_t k = 0;
                            for (uint64_t b = o.shard_index; b < nb_eff; b += shard_count, ++k) {
                                const uint64_t hi = k + 1 < hs.size() ? hs[k + 1] : tot;
                                res->batches.push_back(rpq_batch_info{js[b], js[b + 1], hs[k], hi - hs[k]});
                            }
                        }
                    }
                    res->ncols = 2;
                    res->nrows = tot;
                    if (!dev_alloc_to(res->cols[0], std::max<uint64_t>(tot, 1) * 4, s) ||
                        !dev_alloc_to(res->cols[1], std::max<uint64_t>(tot, 1) * 4, s)) {
                        cudaGetLastError();
                        rpq_result_release(sub_keep);
                        return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (%llu pairs)", (unsigned long long)tot));
                    }
                    k_sparse_thread<false, true><<<grid_for(np), 256, 0, s>>>(A, cand, pidx, np, B, o.shard_index,
                                                                             shard_count, sc, tov, d_stats, start,
                                                                             res->cols[0], res->cols[1]);
                    k_sparse<false, true><<<148 * 8, SP_WARPS * 32, 0, s>>>(A, cand, pidx, tlist, np, B,
                                                                            o.shard_index, shard_count, sc, sov,
                                                                            d_stats, start, res->cols[0],
                                                                            res->cols[1], d_err, d_nt);
                    ST.kernel_launches += 2;
                    if (sub_keep && sub_keep->n_ps) {
                        unsigned long long *ss = (unsigned long long *)ws.get(sub_keep->n_ps * 8);
                        size_t tb3 = 0;
                        cub::DeviceScan::ExclusiveSum(nullptr, tb3, (unsigned long long *)sub_keep->ps_cnt, ss,
                                                      (int64_t)sub_keep->n_ps, s);
                        void *tmp3 = ws.get(tb3);
                        if (!ss || !tmp3) { rpq_result_release(sub_keep); return fail(rpq_fail(RPQ_ENOMEM, "oom")); }
                        cub::DeviceScan::ExclusiveSum(tmp3, tb3, (unsigned long long *)sub_keep->ps_cnt, ss,
                                                      (int64_t)sub_keep->n_ps, s);
                        k_place_sub<<<grid_for(sub_keep->n_ps * 32), 256, 0, s>>>(
                            cand, nsrc, sub_keep->ps_src, (const unsigned long long *)sub_keep->ps_cnt, ss,
                            sub_keep->n_ps, sub_keep->cols[0], sub_keep->cols[1], start, res->cols[0], res->cols[1]);
                        ST.kernel_launches += 2;
                    }
                    if (eps)
                        for (uint64_t b = o.shard_index; b < nb_eff; b += shard_count)
                            if (js[b + 1] > js[b]) {
                                k_write_eps<<<grid_for(js[b + 1] - js[b]), 256, 0, s>>>(
                                    flag, cand, js[b], js[b + 1], start + js[b], res->cols[0], res->cols[1]);
                                ST.kernel_launches++;
                            }
                    int herr = 0;
                    RPQ_CUDA_TRY(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
                    RPQ_CUDA_TRY(cudaStreamSynchronize(s));
                    if (getenv("RPQ_TEST_SPARSE_REDO")) herr = 1;   // test hook: exercise the fallback below
                    rpq_result_release(sub_keep);
                    sub_keep = nullptr;
                    if (herr) {   // rare: redo the whole query on the dense engine
                        rpq_eval_opts d = o;
                        d.reserved |= 1u;
                        rpq_result_release(res);
                        return eval_sources_device(g, a, d_cand_in, nsrc, &d, out);
                    }
                    sparse_total = tot;   // pairs already include epsilon pairs
                }
                sparse_done = true;
                ST.batches += 1;
            }
        }
    }
    // ---- workspace ----------------------------------------------------------
    const uint64_t words = R_max * nw;
    ST.state_words = words;
    const uint64_t nxw = (nchunk + 31) / 32;            // X words per row
    const uint64_t nxwords = R_max * nxw;
    const uint64_t xbwords = (nxwords + 1023) / 1024 + 1;
    const uint32_t hitem_cap = 1u << 14, hrec_cap = 1u << 22;
    uint64_t *Vis = nullptr, *Done = nullptr, *hubF = nullptr;
    uint32_t *X0 = nullptr, *X1 = nullptr, *XB0 = nullptr, *XB1 = nullptr;
    Ctrl *ctrl = (Ctrl *)ws.get(sizeof(Ctrl));
    // small pinned host word for the per-level flag readback (per thread)
    static thread_local uint32_t *h_cnt = nullptr;
    if (!h_cnt) RPQ_CUDA_TRY(cudaMallocHost(&h_cnt, 64));
    HubRec *hrecs = nullptr;
    HubItem *hitems = nullptr;
    uint64_t *N1 = nullptr;
    if (nbatches && !sparse_done) {
        Vis = (uint64_t *)ws.get(words * 8);
        Done = (uint64_t *)ws.get(words * 8);     // bounded: N0
        if (bounded) {
            N1 = (uint64_t *)ws.get(words * 8);
            if (!N1) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (bounded state)"));
            RPQ_CUDA_TRY(cudaMemsetAsync(N1, 0, words * 8, s));
        }
        X0 = (uint32_t *)ws.get(nxwords * 4 + 128);
        X1 = (uint32_t *)ws.get(nxwords * 4 + 128);
        XB0 = (uint32_t *)ws.get(xbwords * 4);
        XB1 = (uint32_t *)ws.get(xbwords * 4);
        hitems = (HubItem *)ws.get((uint64_t)hitem_cap * sizeof(HubItem));
        hubF = (uint64_t *)ws.get((uint64_t)hitem_cap * KGRP * 32 * 8);
        hrecs = (HubRec *)ws.get((uint64_t)hrec_cap * sizeof(HubRec));
        if (!Vis || !Done || !X0 || !X1 || !XB0 || !XB1 || !hitems || !hubF || !hrecs)
            return fail(rpq_fail(RPQ_ENOMEM, "out of device memory for B=%llu sources (%llu state words)",
                                 (unsigned long long)B, (unsigned long long)words));
        RPQ_CUDA_TRY(cudaMemsetAsync(Vis, 0, words * 8, s));
        RPQ_CUDA_TRY(cudaMemsetAsync(Done, 0, words * 8, s));
        RPQ_CUDA_TRY(cudaMemsetAsync(X0, 0, nxwords * 4 + 128, s));
        RPQ_CUDA_TRY(cudaMemsetAsync(X1, 0, nxwords * 4 + 128, s));
        RPQ_CUDA_TRY(cudaMemsetAsync(XB0, 0, xbwords * 4, s));
        RPQ_CUDA_TRY(cudaMemsetAsync(XB1, 0, xbwords * 4, s));
    }
    HM("state alloc+memset");
    if (!ctrl || !d_stats) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory"));
    RPQ_CUDA_TRY(cudaMemsetAsync(ctrl, 0, sizeof(Ctrl), s));

    PT.mark("workspace alloc + clear");
    // per-candidate counts (PER_SOURCE / PAIRS), initialised to the epsilon pair
    if (want_ps && !cand_cnt) {
        cand_cnt = (unsigned long long *)ws.get(std::max<uint64_t>(nsrc, 1) * 8);
        if (!cand_cnt) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (counts)"));
        k_fill_eps<<<grid_for(nsrc), 256, 0, s>>>(cand_cnt, nsrc, eps ? 1ull : 0ull);
        ST.kernel_launches++;
    }
    struct Block { uint32_t *src, *dst; uint64_t n; };
    std::vector<Block> blocks;
    struct BlockGuard { std::vector<Block> *b; cudaStream_t s; ~BlockGuard() { for (auto &x : *b) { dev_free(x.src, s); dev_free(x.dst, s); } } } bgd{&blocks, s};

    uint64_t total = 0;
    // candidate-index interval owned by batch b (non-productive candidates in
    // it contribute their epsilon pair); one virtual batch when P is empty

    // ---- level loop setup: parity-0/1 argument sets and the device graph ----
    Layout *d_layout = (Layout *)ws.get(sizeof(Layout));
    const uint64_t nunits = (nxwords + 31) / 32;
    uint32_t *ulist = (uint32_t *)ws.get((nunits + 1) * 4);
    uint32_t *TX = (uint32_t *)ws.get(nxwords * 4 + 128);
    uint32_t *TU = (uint32_t *)ws.get(((nunits + 31) / 32 + 1) * 4);
    uint32_t *TL = (uint32_t *)ws.get((nunits + 1) * 4);
    if (!d_layout || !ulist || !TX || !TU || !TL) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
    if (nbatches) {
        RPQ_CUDA_TRY(cudaMemsetAsync(TX, 0, nxwords * 4 + 128, s));
        RPQ_CUDA_TRY(cudaMemsetAsync(TU, 0, ((nunits + 31) / 32 + 1) * 4, s));
    }
    LevelArgs P0{}, P1{};
    P0.Vis = Vis; P0.Done = Done;
    P0.Xcur = X0; P0.Xnext = X1; P0.XBcur = XB0; P0.XBnext = XB1;
    P0.nxwords = nxwords;
    P0.ctrl = ctrl; P0.par = 0;
    P0.hitems = hitems; P0.hubF = hubF; P0.hrecs = hrecs;
    P0.hitem_cap = hitem_cap; P0.hrec_cap = hrec_cap;
    P0.nw = (uint32_t)nw; P0.nxw = (uint32_t)nxw; P0.cw = CW;
    P0.stats = d_stats;
    P0.ulist = ulist;
    P0.TX = TX; P0.TU = TU; P0.TL = TL;
    // direction-optimising levels: need the transposed CSR and 32-word chunks
    uint64_t *Act = nullptr;
    {
        uint32_t mode = pull_avail ? 1u : 0u;
        if (CW != 32 || !nbatches || sparse_done || bounded) mode = 0;
        if (mode) {
            Act = (uint64_t *)ws.get(nw * 16);
            if (!Act) mode = 0;
        }
        P0.pull_mode = mode;
        P0.total_units = nunits;
        P0.ActCur = Act;
        P0.ActNext = Act ? Act + nw : nullptr;
    }
    P0.bounded = bounded ? 1u : 0u;
    {   // bulk-copy (TMA) expand: RPQ_TMA=1 (needs 32-word chunks; not with bounded or pull levels)
        // RPQ_TMA = bit 0: k_level, bit 1: k_level_hub (e.g. 1, 2, 3)
        const char *et = getenv("RPQ_TMA");
        const uint32_t tm = et ? (uint32_t)(atoi(et) & 3) : 0u;
        P0.tma = (!bounded && !P0.pull_mode && CW == 32) ? tm : 0u;
        if (P0.tma) {
            static bool attr_set = false;
            if (!attr_set) {
                const void *fns[4] = {(const void *)k_level<false, false, true>, (const void *)k_level<true, false, true>,
                                      (const void *)k_level_hub<false, false, true>,
                                      (const void *)k_level_hub<true, false, true>};
                for (const void *fn : fns)
                    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TMA_SMEM);
                attr_set = true;
            }
        }
    }
    // levels (ctrl->levels, counted from 1) that may expand: level L performs
    // hop L, or hop L + 1 when the seeds were expanded by k_seed_expand
    P0.level_lim = !bounded ? ~0u : skip_q0 ? (max_hops ? max_hops - 1 : 0) : max_hops;
    if (bounded) { P0.Front = Done; P0.Mark = Vis; P0.Disc = N1; }   // N0 = the Done array
    else { P0.Front = Vis; P0.Mark = Done; P0.Disc = Vis; }
    P1 = P0;
    P1.par = 1;
    std::swap(P1.Xcur, P1.Xnext);
    std::swap(P1.XBcur, P1.XBnext);
    std::swap(P1.ActCur, P1.ActNext);
    if (bounded) std::swap(P1.Front, P1.Disc);
    const int lgrid = 148 * RPQ_LEVEL_MINB;   // persistent: warps fetch work units dynamically
    const int hgrid = 148 * RPQ_HUB_MINB;
    // The instantiated level graph is cached per thread and reused when every
    // kernel argument is identical (same automaton, grids and -- thanks to the
    // stream-ordered pool handing back the same blocks -- the same state
    // buffers); otherwise it is rebuilt.  Saves the ~0.1 ms instantiate.
    struct CachedGraph {
        std::vector<unsigned char> key;    // every kernel argument
        std::vector<int> topo;             // kernels / node order
        std::unique_ptr<LevelGraph> lg;
    };
    // (heap object, never destroyed: no graph teardown after the CUDA runtime
    // has shut down at process exit)
    static thread_local CachedGraph &cache = *new CachedGraph();
    LevelGraph local;
    LevelGraph *LGp = &local;
    if (nbatches && !sparse_done && !getenv("RPQ_HOST_LOOP")) {
        std::vector<unsigned char> key;
        auto put = [&](const void *x, size_t n) {
            const unsigned char *b = (const unsigned char *)x;
            key.insert(key.end(), b, b + n);
        };
        int dev = 0;
        cudaGetDevice(&dev);
        const int flags[5] = {dev, lgrid, hgrid, need_hub ? 1 : 0, stats ? 1 : 0};
        put(flags, sizeof(flags));
        put(&xbwords, sizeof(xbwords));
        put(&A, sizeof(A));
        put(&d_layout, sizeof(d_layout));
        put(&P0, sizeof(P0));
        put(&P1, sizeof(P1));
        const std::vector<int> topo = {dev, lgrid, hgrid, need_hub ? 1 : 0, stats ? 1 : 0, bounded ? 1 : 0,
                                       (int)P0.pull_mode, (int)P0.tma};
        bool updated = false;
        if (cache.lg && cache.lg->exec && cache.key == key) {
            LGp = cache.lg.get();
        } else if (cache.lg && cache.lg->exec && cache.topo == topo) {
            // same kernels, new arguments (another graph / state buffers): patch the nodes
            cudaError_t ue =
                stats ? (bounded ? build_level_graph<true, true>(*cache.lg, A, d_layout, P0, P1, lgrid, hgrid, xbwords, need_hub, true)
                                 : build_level_graph<true, false>(*cache.lg, A, d_layout, P0, P1, lgrid, hgrid, xbwords, need_hub, true))
                      : (bounded ? build_level_graph<false, true>(*cache.lg, A, d_layout, P0, P1, lgrid, hgrid, xbwords, need_hub, true)
                                 : build_level_graph<false, false>(*cache.lg, A, d_layout, P0, P1, lgrid, hgrid, xbwords, need_hub, true));
            if (ue == cudaSuccess) {
                cache.key = std::move(key);
                LGp = cache.lg.get();
                updated = true;
            } else {
                cudaGetLastError();
            }
        }
        if (LGp == &local && !updated) {
            cache.lg.reset();
            auto lg = std::make_unique<LevelGraph>();
            cudaError_t ge =
                stats ? (bounded ? build_level_graph<true, true>(*lg, A, d_layout, P0, P1, lgrid, hgrid, xbwords, need_hub)
                                 : build_level_graph<true, false>(*lg, A, d_layout, P0, P1, lgrid, hgrid, xbwords, need_hub))
                      : (bounded ? build_level_graph<false, true>(*lg, A, d_layout, P0, P1, lgrid, hgrid, xbwords, need_hub)
                                 : build_level_graph<false, false>(*lg, A, d_layout, P0, P1, lgrid, hgrid, xbwords, need_hub));
            if (ge != cudaSuccess) {   // fall back to the host-driven loop
                cudaGetLastError();
                if (lg->exec) cudaGraphExecDestroy(lg->exec);
                lg->exec = nullptr;
            } else {
                cache.key = std::move(key);
                cache.topo = topo;
                cache.lg = std::move(lg);
                LGp = cache.lg.get();
            }
        }
    }
    LevelGraph &LG = *LGp;
    PT.mark("level graph");
    HM("level graph");

    // layouts of this shard's batches, computed up front and copied once
    std::vector<Layout> lay_h;
    std::vector<Range> lay_fin, lay_all;
    for (uint64_t b = o.shard_index; b < (sparse_done ? 0 : nbatches); b += shard_count) {
        Layout S{};
        uint64_t rows = 0;
        Range fin_hull{1, 0}, all_hull{1, 0};
        for (uint32_t q = 0; q < a->nq; ++q) {
            Range r = in_range[q];
            if (q == 0 && !skip_q0) r = hull(r, Range{sfirst[b], slast[b]});
            S.row_base[q] = rows;
            S.lo[q] = r.empty() ? 0 : r.lo;
            S.len[q] = r.empty() ? 0 : r.hi - r.lo + 1;
            rows += S.len[q];
            if ((a->final_mask >> q) & 1) fin_hull = hull(fin_hull, r);
            all_hull = hull(all_hull, r);
        }
        lay_h.push_back(S);
        lay_fin.push_back(fin_hull);
        lay_all.push_back(all_hull);
    }
    Layout *d_layouts = (Layout *)ws.get(std::max<size_t>(lay_h.size(), 1) * sizeof(Layout));
    if (!d_layouts) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
    if (!lay_h.empty()) {
        // pageable source: the copy is staged before the call returns
        RPQ_CUDA_TRY(cudaMemcpyAsync(d_layouts, lay_h.data(), lay_h.size() * sizeof(Layout), cudaMemcpyHostToDevice, s));
    }
    RPQ_CUDA_TRY(cudaMemsetAsync(d_total, 0, 8, s));
        HM("layouts");
    size_t lay_i = 0;
    // level-loop timing events (RPQ_TIME_KERNELS), recycled per thread
    static thread_local std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
    auto take_ev = [&]() {
        cudaEvent_t e = nullptr;
        if (!ev_pool.empty()) { e = ev_pool.back(); ev_pool.pop_back(); }
        else cudaEventCreate(&e);
        return e;
    };
    struct TevGuard {
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> *v;
        std::vector<cudaEvent_t> *pool;
        ~TevGuard() { for (auto &e : *v) { pool->push_back(e.first); pool->push_back(e.second); } }
    } tevg{&tev, &ev_pool};
    for (uint64_t b = o.shard_index; b < (sparse_done ? 0 : nb_eff); b += shard_count) {
        const uint64_t jlo = jstart(b), jhi = (b + 1 < nb_eff) ? jstart(b + 1) : nsrc;
        ST.batches++;
        if (b >= nbatches) {   // virtual batch: only epsilon pairs
            const uint64_t ne = eps ? (jhi - jlo) : 0;
            if (want_ps) res->batches.push_back(rpq_batch_info{jlo, jhi, total, ne});
            total += ne;
            if (want_pairs && ne) {
                Block bl{nullptr, nullptr, ne};
                if (!dev_alloc_to(bl.src, ne * 4, s) || !dev_alloc_to(bl.dst, ne * 4, s)) {
                    cudaGetLastError();
                    dev_free(bl.src, s);
                    return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (pairs)"));
                }
                blocks.push_back(bl);
                unsigned long long *start = (unsigned long long *)ws.get(ne * 8 + 8);
                if (!start) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                size_t tb = 0;
                cub::DeviceScan::ExclusiveSum(nullptr, tb, cand_cnt + jlo, start, (int64_t)(jhi - jlo), s);
                void *tmp = ws.get(tb);
                if (!tmp) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
                cub::DeviceScan::ExclusiveSum(tmp, tb, cand_cnt + jlo, start, (int64_t)(jhi - jlo), s);
                k_write_eps<<<grid_for(jhi - jlo), 256, 0, s>>>(flag, cand, jlo, jhi, start, bl.src, bl.dst);
                ST.kernel_launches++;
            }
            continue;
        }
        const uint64_t b0 = b * B;
        const uint32_t nb = (uint32_t)std::min<uint64_t>(B, np - b0);
        const Layout &S = lay_h[lay_i];
        const Range fin_hull = lay_fin[lay_i];
        if (lay_i > 0) {   // clear what the previous batch of this shard touched
            k_clear_touched<<<148 * 8, 256, 0, s>>>(P0, nunits, dead_final);
            k_clear_dense<<<148 * 8, 256, 0, s>>>(Vis, Done, words, TX, nxwords + 32, TU, (nunits + 31) / 32 + 1,
                                                  ctrl, nunits, dead_final);
            ST.kernel_launches += 2;
        }
        RPQ_CUDA_TRY(cudaMemcpyAsync(d_layout, d_layouts + lay_i, sizeof(Layout), cudaMemcpyDeviceToDevice, s));
        ++lay_i;
        if (Act) RPQ_CUDA_TRY(cudaMemsetAsync(Act, 0, nw * 16, s));
        // seeds: into Vis, or (bounded) into N0, the first level's frontier
        k_seed<<<grid_for(nb), 256, 0, s>>>(S, cand, pidx, b0, nb, bounded ? Done : Vis, X0, XB0, (uint32_t)nw,
                                            (uint32_t)nxw, CW, ctrl, skip_q0 ? 1 : 0, Act);
        ST.kernel_launches++;
        if (skip_q0 && (!bounded || max_hops >= 1)) {
            const int sg = grid_for((uint64_t)nb * 32, 256, 148 * 8);
            const int seed_lanes = getenv("RPQ_SEED_WARPS") ? 0 : 1;
            if (seed_lanes) k_seed_lanes<<<grid_for(nb), 256, 0, s>>>(A, d_layout, P1, cand, pidx, b0, nb);
            if (stats && bounded) {
                k_seed_expand<true, true><<<sg, 256, 0, s>>>(A, d_layout, P1, cand, pidx, b0, nb, seed_lanes);
                if (need_hub) k_level_hub<true, true><<<hgrid, 256, 0, s>>>(A, d_layout, P1);
            } else if (stats) {
                k_seed_expand<true><<<sg, 256, 0, s>>>(A, d_layout, P1, cand, pidx, b0, nb, seed_lanes);
                if (need_hub) k_level_hub<true><<<hgrid, 256, 0, s>>>(A, d_layout, P1);
            } else if (bounded) {
                k_seed_expand<false, true><<<sg, 256, 0, s>>>(A, d_layout, P1, cand, pidx, b0, nb, seed_lanes);
                if (need_hub) k_level_hub<false, true><<<hgrid, 256, 0, s>>>(A, d_layout, P1);
            } else {
                k_seed_expand<false><<<sg, 256, 0, s>>>(A, d_layout, P1, cand, pidx, b0, nb, seed_lanes);
                if (need_hub) k_level_hub<false><<<hgrid, 256, 0, s>>>(A, d_layout, P1);
            }
            if (seed_lanes) k_xb_from_x<<<grid_for(nxwords, 256, 148 * 8), 256, 0, s>>>(X0, nxwords, XB0);
            ST.kernel_launches += (need_hub ? 2 : 1) + (seed_lanes ? 2 : 0);
        }
        PT.mark("seed");
        rpq_status st = RPQ_OK;
        if (timeit) {
            tev.emplace_back(take_ev(), take_ev());
            cudaEventRecord(tev.back().first, s);
        }
        if (LG.exec) {
            cudaError_t ge = cudaGraphLaunch(LG.exec, s);
            if (ge != cudaSuccess) st = rpq_fail(RPQ_ECUDA, "cudaGraphLaunch: %s", cudaGetErrorString(ge));
        } else {
            st = run_levels_host(A, d_layout, P0, P1, lgrid, hgrid, xbwords, s, stats, h_cnt, &ST, need_hub);
        }
        if (timeit) cudaEventRecord(tev.back().second, s);
        PT.mark("levels");
        HM("levels enqueued");
        if (st != RPQ_OK) return fail(st);
        // bounded: the loop may have stopped with activity left (levels past
        // the bound return at once): clear the bitmaps for the next batch
        if (bounded) {
            RPQ_CUDA_TRY(cudaMemsetAsync(X0, 0, nxwords * 4 + 128, s));
            RPQ_CUDA_TRY(cudaMemsetAsync(X1, 0, nxwords * 4 + 128, s));
            RPQ_CUDA_TRY(cudaMemsetAsync(XB0, 0, xbwords * 4, s));
            RPQ_CUDA_TRY(cudaMemsetAsync(XB1, 0, xbwords * 4, s));
        }
        // (bounded: Vis holds exactly the expanded bits (depth < bound) until
        // k_merge_bounded below adds the last level's; PE is taken before)
        if (want_spe) {   // per-source PE of this batch -> cand_pe
            unsigned long long *bpe = (unsigned long long *)ws.get((uint64_t)nb * 8);
            if (!bpe) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
            RPQ_CUDA_TRY(cudaMemsetAsync(bpe, 0, (uint64_t)nb * 8, s));
            k_source_pe<<<148 * 8, 256, 0, s>>>(A, S, Vis, (uint32_t)nw, nb, bpe);
            if (skip_q0 && (!bounded || max_hops >= 1))
                k_source_pe_seeds<<<grid_for(nb), 256, 0, s>>>(A, cand, pidx, b0, nb, bpe);
            k_scatter_counts<<<grid_for(nb), 256, 0, s>>>(bpe, pidx, b0, nb, cand_pe);
            ST.kernel_launches += skip_q0 ? 3 : 2;
        }
        if (want_pe) {   // PE after the fact (exact for push and pull levels alike)
            const bool rows = want_ps || bounded;   // else fused into the count pass
            const bool seeds = skip_q0 && (!bounded || max_hops >= 1);
            if (rows) k_pe_rows<<<148 * 8, 256, 0, s>>>(A, S, Vis, (uint32_t)nw, d_stats + S_PE_POST);
            if (seeds) k_pe_seeds<<<grid_for(nb), 256, 0, s>>>(A, cand, pidx, b0, nb, d_stats + S_PE_POST);
            ST.kernel_launches += (rows ? 1 : 0) + (seeds ? 1 : 0);
        }
        if (bounded) {
            k_merge_bounded<<<148 * 8, 256, 0, s>>>(Vis, Done, N1, words);
            ST.kernel_launches++;
        }
        // X and XB are all zero again here (the last level activated
        // nothing).  Extraction reads Vis of the final states.
        const uint32_t vlo = fin_hull.empty() ? 0 : fin_hull.lo;
        const uint64_t vn = fin_hull.empty() ? 0 : (uint64_t)fin_hull.hi - fin_hull.lo + 1;
        const uint64_t eps_np = eps ? (jhi - jlo) - nb : 0;   // non-productive candidates in the interval
        if (!want_ps) {
            // COUNT: accumulate on the device (sparse or dense path chosen
            // there from the touched-unit count); no host round trip.  With
            // PE the count pass reads every state's rows (hull of all ranges).
            const Range all_hull = lay_all[lay_i - 1];
            const bool fuse_pe = want_pe && !bounded;
            const uint32_t clo = fuse_pe ? (all_hull.empty() ? 0 : all_hull.lo) : vlo;
            const uint64_t cn = fuse_pe ? (all_hull.empty() ? 0 : (uint64_t)all_hull.hi - all_hull.lo + 1) : vn;
            unsigned long long *pe_out = (want_pe && !bounded) ? d_stats + S_PE_POST : nullptr;
            k_count_touched<<<148 * 8, 256, 0, s>>>(A, S, P0, nunits, d_total, dead_final, pe_out);
            if (cn) k_count_total<<<grid_for(cn * 32), 256, 0, s>>>(A, S, Vis, clo, cn, (uint32_t)nw, d_total, ctrl,
                                                                     nunits, nxwords, dead_final, pe_out);
            ST.kernel_launches += cn ? 2 : 1;
            total += eps_np;
            continue;
        }
        const uint32_t nseg = (uint32_t)std::max<uint64_t>(1, (vn + TILE_V - 1) / TILE_V);
        uint32_t *cnt = (uint32_t *)ws.get((uint64_t)nb * nseg * 4);
        unsigned long long *tot = (unsigned long long *)ws.get((uint64_t)nb * 8);
        if (!cnt || !tot) return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (extraction)"));
        RPQ_CUDA_TRY(cudaMemsetAsync(cnt, 0, (uint64_t)nb * nseg * 4, s));
        // tile tasks: parts of tpp tiles x groups of 4 words (k_tile_counts, k_write_pairs)
        const uint64_t nwg = (nw + 3) / 4;
        const uint64_t nparts = std::min<uint64_t>(nseg, ((uint64_t)148 * 6 * 4 + nwg - 1) / nwg);
        const uint32_t tpp = (uint32_t)((nseg + nparts - 1) / nparts);
        const uint64_t ntask = nwg * ((nseg + tpp - 1) / tpp);
        if (vn) {
            k_tile_counts<<<(unsigned)std::min<uint64_t>(ntask, 148 * 12), 128, 0, s>>>(A, S, Vis, vlo, vn,
                                                                                     (uint32_t)nw, nb, nseg, tpp, cnt);
            ST.kernel_launches++;
        }
        k_row_scan<<<grid_for((uint64_t)nb * 32), 256, 0, s>>>(cnt, nb, nseg, tot);
        k_scatter_counts<<<grid_for(nb), 256, 0, s>>>(tot, pidx, b0, nb, cand_cnt);
        ST.kernel_launches += 2;
        // start offsets of every candidate in [jlo, jhi)
        const uint64_t nj = jhi - jlo;
        unsigned long long *start = (unsigned long long *)ws.get((nj + 1) * 8);
        if (!start) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, cand_cnt + jlo, start, (int64_t)nj, s);
        void *tmp = ws.get(tb);
        if (!tmp) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
        cub::DeviceScan::ExclusiveSum(tmp, tb, cand_cnt + jlo, start, (int64_t)nj, s);
        unsigned long long last_start = 0, last_cnt = 0;
        RPQ_CUDA_TRY(cudaMemcpyAsync(&last_start, start + nj - 1, 8, cudaMemcpyDeviceToHost, s));
        RPQ_CUDA_TRY(cudaMemcpyAsync(&last_cnt, cand_cnt + jhi - 1, 8, cudaMemcpyDeviceToHost, s));
        RPQ_CUDA_TRY(cudaStreamSynchronize(s));
        const uint64_t bt = last_start + last_cnt;
        res->batches.push_back(rpq_batch_info{jlo, jhi, total, bt});
        total += bt;
        if (want_pairs && bt) {
            Block bl{nullptr, nullptr, bt};
            HM("pairs: count + scan");
            if (!dev_alloc_to(bl.src, bt * 4, s) || !dev_alloc_to(bl.dst, bt * 4, s)) {
                cudaGetLastError();
                dev_free(bl.src, s);
                return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (%llu pairs)", (unsigned long long)bt));
            }
            blocks.push_back(bl);
            HM("pairs: cudaMalloc of the block");
            if (vn) {
                k_write_pairs<<<(unsigned)std::min<uint64_t>(ntask, 148 * 6), WP_WARPS * 32, 0, s>>>(
                    A, S, Vis, vlo, vn, (uint32_t)nw, nb, nseg, tpp, cnt, cand, pidx, b0, start, jlo, bl.src, bl.dst);
                ST.kernel_launches++;
            }
            if (eps) {
                k_write_eps<<<grid_for(nj), 256, 0, s>>>(flag, cand, jlo, jhi, start, bl.src, bl.dst);
                ST.kernel_launches++;
            }
        }
        RPQ_CUDA_TRY(cudaGetLastError());
    }

    if (sparse_done) total = sparse_total;
    // everything the host still needs (device COUNT total, |listed sources|,
    // level counter, statistics) comes back in ONE synchronisation at the end
    struct Fin {
        unsigned long long total;
        uint64_t n_ps;
        Ctrl ctrl;
        unsigned long long hs[NSTAT];
    };
    static thread_local Fin *fin = nullptr;
    if (!fin) RPQ_CUDA_TRY(cudaMallocHost(&fin, sizeof(Fin)));
    memset(fin, 0, sizeof(Fin));
    const bool dev_total = !want_ps && nbatches && !sparse_done;
    if (dev_total) RPQ_CUDA_TRY(cudaMemcpyAsync(&fin->total, d_total, 8, cudaMemcpyDeviceToHost, s));
    PT.mark("extraction");
    HM("extraction+readback");
    // ---- result assembly ---------------------------------------------------
    res->count = total;
    if (want_pairs && !sparse_done) {
        res->ncols = 2;
        res->nrows = total;
        if (blocks.size() == 1) {
            res->cols[0] = blocks[0].src;
            res->cols[1] = blocks[0].dst;
            blocks.clear();
        } else {
            if (!dev_alloc_to(res->cols[0], std::max<uint64_t>(total, 1) * 4, s) ||
                !dev_alloc_to(res->cols[1], std::max<uint64_t>(total, 1) * 4, s)) {
                cudaGetLastError();
                return fail(rpq_fail(RPQ_ENOMEM, "out of device memory (pairs)"));
            }
            uint64_t off = 0;
            for (auto &bl : blocks) {
                RPQ_CUDA_TRY(cudaMemcpyAsync(res->cols[0] + off, bl.src, bl.n * 4, cudaMemcpyDeviceToDevice, s));
                RPQ_CUDA_TRY(cudaMemcpyAsync(res->cols[1] + off, bl.dst, bl.n * 4, cudaMemcpyDeviceToDevice, s));
                off += bl.n;
            }
        }
    }
    if (want_ps && nsrc) {
        // non-zero (source, count) of this shard's batches, ascending source.
        // Candidates of other shards' batches are zeroed first.
        std::vector<std::pair<uint64_t, uint64_t>> foreign;
        for (uint64_t b = 0; b < nb_eff; ++b)
            if (b % shard_count != o.shard_index) {
                uint64_t jl = jstart(b), jh = (b + 1 < nb_eff) ? jstart(b + 1) : nsrc;
                if (jh > jl) RPQ_CUDA_TRY(cudaMemsetAsync(cand_cnt + jl, 0, (jh - jl) * 8, s));
                if (jh > jl && want_spe) RPQ_CUDA_TRY(cudaMemsetAsync(cand_pe + jl, 0, (jh - jl) * 8, s));
            }
        uint8_t *nz = (uint8_t *)ws.get(nsrc);
        uint64_t *d_n = (uint64_t *)ws.get(8);
        if (!nz || !d_n) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
        if (!dev_alloc_to(res->ps_src, nsrc * 4, s) || !dev_alloc_to(res->ps_cnt, nsrc * 8, s)) {
            cudaGetLastError();
            return fail(rpq_fail(RPQ_ENOMEM, "oom"));
        }
        if (want_spe && !dev_alloc_to(res->ps_pe, nsrc * 8, s)) {
            cudaGetLastError();
            return fail(rpq_fail(RPQ_ENOMEM, "oom"));
        }
        // listed: non-zero count (or, with RPQ_SOURCE_PE, non-zero PE)
        k_ps_flags<<<grid_for(nsrc), 256, 0, s>>>(cand_cnt, want_spe ? cand_pe : nullptr, nsrc, nz);
        size_t tb1 = 0, tb2 = 0;
        cub::DeviceSelect::Flagged(nullptr, tb1, cand_cnt, nz, (unsigned long long *)res->ps_cnt, d_n, (int64_t)nsrc, s);
        cub::DeviceSelect::Flagged(nullptr, tb2, cand, nz, res->ps_src, d_n, (int64_t)nsrc, s);
        void *tmp = ws.get(std::max(tb1, tb2));
        if (!tmp) return fail(rpq_fail(RPQ_ENOMEM, "oom"));
        cub::DeviceSelect::Flagged(tmp, tb1, cand_cnt, nz, (unsigned long long *)res->ps_cnt, d_n, (int64_t)nsrc, s);
        if (want_spe)
            cub::DeviceSelect::Flagged(tmp, tb1, cand_pe, nz, (unsigned long long *)res->ps_pe, d_n, (int64_t)nsrc, s);
        cub::DeviceSelect::Flagged(tmp, tb2, cand, nz, res->ps_src, d_n, (int64_t)nsrc, s);
        RPQ_CUDA_TRY(cudaMemcpyAsync(&fin->n_ps, d_n, 8, cudaMemcpyDeviceToHost, s));
    }
    if (nbatches && !sparse_done) RPQ_CUDA_TRY(cudaMemcpyAsync(&fin->ctrl, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    if (stats || want_pe) RPQ_CUDA_TRY(cudaMemcpyAsync(fin->hs, d_stats, sizeof(fin->hs), cudaMemcpyDeviceToHost, s));
    cudaEventRecord(e_end, s);
    RPQ_CUDA_TRY(cudaStreamSynchronize(s));
    if (dev_total) {
        total += fin->total;
        res->count = total;
    }
    if (want_ps && nsrc) res->n_ps = fin->n_ps;
    for (auto &e : tev) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e.first, e.second);
        ST.expand_ms += ms;
    }
    if (nbatches && !sparse_done) {
        const Ctrl &hc = fin->ctrl;
        ST.levels = hc.levels;
        if (LG.exec)
            ST.kernel_launches += (2ull + (need_hub ? 1 : 0) + (P0.pull_mode ? 2 : 0)) * hc.levels + (hc.levels + 1) / 2;
        ST.expand_launches = 2ull * ST.levels;
    }
    if (stats || want_pe) {
        const unsigned long long *hs = fin->hs;
        // dense batches: PE after the fact (k_pe_rows/k_pe_seeds); the sparse
        // tiers count it per source (S_PE)
        ST.product_edges = hs[S_PE_POST] + (sparse_done ? hs[S_PE] : 0ull) + sub_pe;
        ST.pull_levels = hs[S_PULL_LEVELS];
        ST.pull_loads = hs[S_PULL_LOADS];
        ST.pull_words = hs[S_PULL_WORDS];
        ST.adv_words = hs[S_ADV_WORDS];
        ST.adv_zero_sectors = hs[S_ADV_ZERO_SECTORS];
        ST.word_items = hs[S_WORD_ITEMS];
        ST.word_edge_ops = hs[S_WORD_EDGE];
        ST.items = hs[S_ITEMS];
        ST.item_edges = hs[S_ITEM_EDGES];
        ST.item_transitions = hs[S_ITEM_TRANS];
        ST.activations = hs[S_X_RED];
        ST.next_reds = hs[S_N_RED];
    }
    float tms = 0;
    cudaEventElapsedTime(&tms, e_begin, e_end);
    ST.total_ms = tms;
    PT.mark("assembly");
    HM("assembly");
    RPQ_CUDA_TRY(cudaGetLastError());
    *out = res;
    return RPQ_OK;
}

// The automatic batch width comes from a cached free-memory figure; if the
// evaluation runs out of memory under it, refresh the figure and retry once.
rpq_status eval_sources_device(const rpq_graph *g, const rpq_nfa *a, const uint32_t *d_cand_in, uint64_t nsrc,
                               const rpq_eval_opts *opts_in, rpq_result **out) {
    bool cached = false;
    rpq_status st = eval_sources_impl(g, a, d_cand_in, nsrc, opts_in, out, &cached);
    if (st == RPQ_ENOMEM && cached) {
        dev_available_invalidate();
        st = eval_sources_impl(g, a, d_cand_in, nsrc, opts_in, out, &cached);
    }
    return st;
}

// ---- public entry points ----------------------------------------------------
static rpq_status check_common(const rpq_graph *g, const rpq_nfa *a, rpq_result **out) {
    if (out) *out = nullptr;
    if (!g || !a || !out) return rpq_fail(RPQ_EINVAL, "NULL argument");
    return RPQ_OK;
}

extern "C" rpq_status rpq_eval_allpairs(const rpq_graph *g, const rpq_nfa *a, const rpq_eval_opts *opts,
                                        rpq_result **out) {
    NvtxRange nvtx_("rpq_eval_allpairs");
    rpq_status st = check_common(g, a, out);
    if (st) return st;
    return eval_sources_device(g, a, nullptr, 0, opts, out);
}

extern "C" rpq_status rpq_plan(const rpq_graph *g, const rpq_nfa *a, const rpq_eval_opts *opts,
                               rpq_plan_info *info) {
    NvtxRange nvtx_("rpq_plan");
    if (!g || !a || !info) return rpq_fail(RPQ_EINVAL, "NULL argument");
    rpq_eval_opts o{};
    if (opts) o = *opts;
    o.reserved |= 4u;
    rpq_result *r = nullptr;
    rpq_status st = eval_sources_device(g, a, nullptr, 0, &o, &r);
    if (st != RPQ_OK) return st;
    info->productive_sources = r->stats.productive_sources;
    info->batch_sources = r->stats.batch_sources;
    info->num_batches = r->stats.batches;
    info->state_words = r->stats.state_words;
    info->chunk_words = r->stats.chunk_words;
    rpq_result_release(r);
    return RPQ_OK;
}

extern "C" rpq_status rpq_eval_sources(const rpq_graph *g, const rpq_nfa *a, const uint32_t *srcs, uint64_t n,
                                       const rpq_eval_opts *opts, rpq_result **out) {
    NvtxRange nvtx_("rpq_eval_sources");
    rpq_status st = check_common(g, a, out);
    if (st) return st;
    if (n && !srcs) return rpq_fail(RPQ_EINVAL, "NULL sources");
    std::vector<uint32_t> v(srcs, srcs + n);
    std::sort(v.begin(), v.end());
    for (uint64_t i = 0; i < n; ++i) {
        if (v[i] >= g->nv) return rpq_fail(RPQ_EINVAL, "source %u >= |V| = %u", v[i], g->nv);
        if (i && v[i] == v[i - 1]) return rpq_fail(RPQ_EINVAL, "duplicate source %u", v[i]);
    }
    RPQ_CUDA_TRY(cudaSetDevice(g->device));
    cudaStream_t s = opts ? (cudaStream_t)opts->cuda_stream : nullptr;
    uint32_t *d = (uint32_t *)dev_alloc(std::max<uint64_t>(n, 1) * 4, s);
    if (!d) return rpq_fail(RPQ_ENOMEM, "out of device memory");
    if (n) {
        cudaError_t e = cudaMemcpyAsync(d, v.data(), n * 4, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) { dev_free(d, s); return rpq_fail(RPQ_ECUDA, "%s", cudaGetErrorString(e)); }
    }
    st = eval_sources_device(g, a, d, n, opts, out);
    dev_free(d, s);
    return st;
}

extern "C" rpq_status rpq_eval_allpairs_stream(const rpq_graph *g, const rpq_nfa *a, const rpq_eval_opts *opts,
                                               uint64_t device_budget_bytes, uint64_t piece_pairs,
                                               rpq_pairs_sink sink, void *ctx, uint64_t *total) {
    NvtxRange nvtx_("rpq_eval_allpairs_stream");
    if (total) *total = 0;
    rpq_result *dummy = nullptr;
    rpq_status st = check_common(g, a, &dummy);
    if (st) return st;
    if (!sink) return rpq_fail(RPQ_EINVAL, "rpq_eval_allpairs_stream: NULL sink");
    rpq_eval_opts o{};
    if (opts) o = *opts;
    const uint32_t shard_count = o.shard_count ? o.shard_count : 1;
    if (o.shard_index >= shard_count) return rpq_fail(RPQ_EINVAL, "shard_index >= shard_count");
    // chunk boundaries follow the device budget: ranks must pass the same one
    if (shard_count > 1 && !device_budget_bytes)
        return rpq_fail(RPQ_EINVAL, "sharded streaming needs an explicit device_budget_bytes (same on every rank)");
    RPQ_CUDA_TRY(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)o.cuda_stream;
    if (!piece_pairs) piece_pairs = 1ull << 26;
    // (1) output size per source: one PER_SOURCE pass over all of V
    rpq_eval_opts po = o;
    po.mode = RPQ_PER_SOURCE;
    po.shard_index = 0;
    po.shard_count = 1;
    rpq_result *pr = nullptr;
    if ((st = eval_sources_device(g, a, nullptr, 0, &po, &pr)) != RPQ_OK) return st;
    std::vector<uint32_t> ps(pr->n_ps);
    std::vector<uint64_t> pc(pr->n_ps);
    if (pr->n_ps) {
        cudaMemcpy(ps.data(), pr->ps_src, pr->n_ps * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(pc.data(), pr->ps_cnt, pr->n_ps * 8, cudaMemcpyDeviceToHost);
    }
    rpq_result_release(pr);
    RPQ_CUDA_TRY(cudaGetLastError());
    // (2) chunks of consecutive sources whose pairs fit the device budget
    if (!device_budget_bytes) device_budget_bytes = dev_available() / 4;
    const uint64_t cap = std::max<uint64_t>(device_budget_bytes / 8, 1);
    std::vector<uint32_t> cstart{0};
    uint64_t acc = 0;
    for (size_t i = 0; i < ps.size(); ++i) {
        if (acc && acc + pc[i] > cap) { cstart.push_back(ps[i]); acc = 0; }
        acc += pc[i];
    }
    cstart.push_back(g->nv);
    // (3) per chunk: PAIRS on the device, pieces through pinned buffers
    uint32_t *h[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    struct Cleanup {
        uint32_t *(*h)[2]; cudaStream_t *cs; cudaEvent_t *ev;
        ~Cleanup() {
            for (int b = 0; b < 2; ++b) for (int c = 0; c < 2; ++c) if (h[b][c]) cudaFreeHost(h[b][c]);
            for (int b = 0; b < 2; ++b) if (ev[b]) cudaEventDestroy(ev[b]);
            if (*cs) cudaStreamDestroy(*cs);
        }
    } cl{h, &cs, ev};
    for (int b = 0; b < 2; ++b)
        for (int c = 0; c < 2; ++c) RPQ_CUDA_TRY(cudaMallocHost(&h[b][c], piece_pairs * 4));
    RPQ_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) RPQ_CUDA_TRY(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    uint64_t delivered = 0;
    rpq_eval_opts co = o;
    co.mode = RPQ_PAIRS | (o.mode & (RPQ_STATS | RPQ_TIME_KERNELS));
    co.shard_index = 0;
    co.shard_count = 1;
    for (size_t c = 0; c + 1 < cstart.size(); ++c) {
        if (c % shard_count != o.shard_index) continue;
        const uint32_t v0 = cstart[c], v1 = cstart[c + 1];
        uint32_t *d = (uint32_t *)dev_alloc((uint64_t)(v1 - v0) * 4, s);
        if (!d) return rpq_fail(RPQ_ENOMEM, "out of device memory (stream chunk)");
        k_iota<<<grid_for(v1 - v0), 256, 0, s>>>(d, v1 - v0);
        k_add_const<<<grid_for(v1 - v0), 256, 0, s>>>(d, v1 - v0, v0);
        rpq_result *r = nullptr;
        st = eval_sources_device(g, a, d, v1 - v0, &co, &r);
        dev_free(d, s);
        if (st != RPQ_OK) return st;
        struct RG { rpq_result *r; ~RG() { rpq_result_release(r); } } rg{r};
        const uint64_t n = r->nrows;
        const uint64_t npieces = (n + piece_pairs - 1) / piece_pairs;
        auto issue = [&](uint64_t k) -> cudaError_t {
            const uint64_t o0 = k * piece_pairs, m = std::min<uint64_t>(piece_pairs, n - o0);
            const int b = (int)(k & 1);
            cudaError_t e = cudaMemcpyAsync(h[b][0], r->cols[0] + o0, m * 4, cudaMemcpyDeviceToHost, cs);
            if (e == cudaSuccess) e = cudaMemcpyAsync(h[b][1], r->cols[1] + o0, m * 4, cudaMemcpyDeviceToHost, cs);
            if (e == cudaSuccess) e = cudaEventRecord(ev[b], cs);
            return e;
        };
        if (npieces) RPQ_CUDA_TRY(issue(0));
        for (uint64_t k = 0; k < npieces; ++k) {
            const int b = (int)(k & 1);
            RPQ_CUDA_TRY(cudaEventSynchronize(ev[b]));
            if (k + 1 < npieces) RPQ_CUDA_TRY(issue(k + 1));   // overlaps the sink below
            const uint64_t m = std::min<uint64_t>(piece_pairs, n - k * piece_pairs);
            const int stop = sink(h[b][0], h[b][1], m, ctx);
            delivered += m;
            if (stop) {
                cudaStreamSynchronize(cs);
                if (total) *total = delivered;
                return RPQ_OK;
            }
        }
    }
    if (total) *total = delivered;
    return RPQ_OK;
}

// Loop-cache plan (WavePlan A2: "partial query results are first
// materialized ... and then reused in subsequent RPQ exploration"): R(inner)
// over all of V, installed in the graph as the derived label `name`, so that
// e.g. a (b c)* d runs as a L? d with L = R((b c)+).
extern "C" rpq_status rpq_cache_closure(rpq_graph *g, const rpq_nfa *inner, const char *name,
                                        const rpq_eval_opts *opts, uint32_t *label_id) {
    NvtxRange nvtx_("rpq_cache_closure");
    rpq_result *r = nullptr;
    rpq_status st = check_common(g, inner, &r);
    if (st) return st;
    rpq_eval_opts o{};
    if (opts) o = *opts;
    o.mode = RPQ_PAIRS | (o.mode & (RPQ_STATS | RPQ_TIME_KERNELS | RPQ_BOUNDED));
    o.shard_index = 0;
    o.shard_count = 1;
    if ((st = eval_sources_device(g, inner, nullptr, 0, &o, &r)) != RPQ_OK) return st;
    st = rpq_graph_add_label(g, name, r->cols[0], r->cols[1], r->nrows, 1, o.cuda_stream, label_id);
    rpq_result_release(r);
    return st;
}

// The whole loop-cache plan for all-pairs R(prefix (loop)* suffix): cache
// R(loop+) as a fresh derived label L, then evaluate "(prefix) L? (suffix)".
extern "C" rpq_status rpq_eval_loop_cached(rpq_graph *g, const char *prefix, const char *loop, const char *suffix,
                                           const rpq_eval_opts *opts, rpq_result **out) {
    NvtxRange nvtx_("rpq_eval_loop_cached");
    if (out) *out = nullptr;
    if (!g || !loop || !out) return rpq_fail(RPQ_EINVAL, "rpq_eval_loop_cached: NULL argument");
    static std::atomic<uint32_t> next_id{0};
    std::string name;
    for (;;) {   // a label name not in the vocabulary
        name = "__loop" + std::to_string(next_id++);
        if (std::find(g->label_names.begin(), g->label_names.end(), name) == g->label_names.end()) break;
    }
    rpq_nfa *inner = nullptr, *outer = nullptr;
    struct G2 { rpq_nfa **a, **b; ~G2() { delete *a; delete *b; } } gd{&inner, &outer};
    size_t eo = 0;
    const std::string lp = "(" + std::string(loop) + ")+";
    rpq_status st = compile_regex(g->label_names, lp.c_str(), 0, &inner, &eo);
    if (st != RPQ_OK) return st;
    rpq_eval_opts co{};
    if (opts) co = *opts;
    co.mode &= ~(uint32_t)RPQ_BOUNDED;   // the closure itself is unbounded
    if ((st = rpq_cache_closure(g, inner, name.c_str(), &co, nullptr)) != RPQ_OK) return st;
    auto blank = [](const char *x) {
        if (!x) return true;
        for (; *x; ++x) if (!isspace((unsigned char)*x)) return false;
        return true;
    };
    std::string q;
    if (!blank(prefix)) q += "(" + std::string(prefix) + ") ";
    q += name + "?";
    if (!blank(suffix)) q += " (" + std::string(suffix) + ")";
    if ((st = compile_regex(g->label_names, q.c_str(), 0, &outer, &eo)) != RPQ_OK) return st;
    return rpq_eval_allpairs(g, outer, opts, out);
}

extern "C" rpq_status rpq_eval_targets(const rpq_graph *g, const rpq_nfa *a, const uint32_t *targets,
                                       uint64_t n, const rpq_eval_opts *opts, rpq_result **out) {
    NvtxRange nvtx_("rpq_eval_targets");
    rpq_status st = check_common(g, a, out);
    if (st) return st;
    if (g->in_csr.size() != g->csr.size())
        return rpq_fail(RPQ_EUNSUPPORTED, "rpq_eval_targets: graph loaded without RPQ_GRAPH_IN_EDGES");
    rpq_nfa *rev = nullptr;
    if ((st = reverse_automaton(a, &rev)) != RPQ_OK) return st;
    struct NfaGuard { rpq_nfa *p; ~NfaGuard() { delete p; } } ng{rev};
    rpq_eval_opts o{};
    if (opts) o = *opts;
    o.reserved |= 2u;
    // (t, x) pairs of rho^R on the transposed graph, sorted by (t, x)
    if ((st = rpq_eval_sources(g, rev, targets, n, &o, out)) != RPQ_OK) return st;
    rpq_result *r = *out;
    if (r->ncols == 2) std::swap(r->cols[0], r->cols[1]);   // -> (x, t) columns
    return RPQ_OK;
}

extern "C" rpq_status rpq_eval_single_target(const rpq_graph *g, const rpq_nfa *a, uint32_t t,
                                             const rpq_eval_opts *opts, rpq_result **out) {
    rpq_status st = check_common(g, a, out);
    if (st) return st;
    if (t >= g->nv) return rpq_fail(RPQ_EINVAL, "target %u >= |V| = %u", t, g->nv);
    return rpq_eval_targets(g, a, &t, 1, opts, out);
}

extern "C" rpq_status rpq_eval_single_source(const rpq_graph *g, const rpq_nfa *a, uint32_t src,
                                             const rpq_eval_opts *opts, rpq_result **out) {
    rpq_status st = check_common(g, a, out);
    if (st) return st;
    if (src >= g->nv) return rpq_fail(RPQ_EINVAL, "source %u >= |V| = %u", src, g->nv);
    return rpq_eval_sources(g, a, &src, 1, opts, out);
}
