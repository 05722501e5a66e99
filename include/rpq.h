/*
 * include/rpq.h -- C-ABI of the B200-native RPQ / CRPQ hot path.
 *
 * Citations: PAPER.md = /root/reference/PAPER.md (cuRPQ, arXiv 2602.20748),
 * "P:n" = line n.  SURVEY.md §8(b) lists these calls; DESIGN.md gives the
 * readings (R1..R19) referred to below.
 *
 * Conventions (all functions):
 *   - Return rpq_status (0 = OK, < 0 = error); nothing throws across the ABI.
 *     On error every output handle is set to NULL and rpq_last_error() holds a
 *     thread-local message.
 *   - Inputs are caller-owned and copied (host arrays) or only read during
 *     the call (device arrays).  Handles are library-owned and released by the
 *     matching *_free.
 *   - There is no CPU fallback: a call that needs the GPU returns RPQ_ECUDA
 *     when no CUDA device is usable.  Only rpq_compile_labels, the rpq_nfa_*
 *     queries and rpq_last_error run without a GPU.
 *   - Vertex ids are u32 in [0, num_vertices) (vertex v_i has id i).
 *   - Graphs and automata are immutable after creation; concurrent
 *     evaluations on different streams may share them.
 */
#ifndef RPQ_H
#define RPQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RPQ_OK = 0,
    RPQ_EINVAL = -1,        /* bad argument / data (vertex id >= |V|, duplicate source, NULL) */
    RPQ_ESYNTAX = -2,       /* regex syntax error (err_offset = byte offset) */
    RPQ_ELABEL = -3,        /* regex names a label not in the vocabulary */
    RPQ_ENOMEM = -4,        /* device or host allocation failed / budget too small */
    RPQ_ECUDA = -5,         /* CUDA error or no usable device */
    RPQ_ECAPACITY = -6,     /* caller buffer too small (required size returned) */
    RPQ_EUNSUPPORTED = -7   /* automaton too large, disconnected CRPQ, ... */
} rpq_status;

typedef struct rpq_graph rpq_graph;
typedef struct rpq_nfa rpq_nfa;
typedef struct rpq_result rpq_result;

/* ------------------------------------------------------------------------
 * Graph: G = (V, E, L) with labelled vertices and edges.
 * E is a SET of (u, label, w) triples (reading R4): duplicates collapse at
 * load; self-loops are 1-hop paths (R5).  The device layout is one CSR per
 * edge label ("a separate grid is maintained for each edge label"):
 * off_l[|V|+1] (u32) and nbr_l[] (u32, ascending per row, 256-byte aligned
 * base so rows can be read with 128-bit loads), plus the per-label
 * [min, max] of source and destination ids.
 * ------------------------------------------------------------------------ */
typedef struct {
    uint32_t num_vertices;
    uint64_t num_edges;
    const uint32_t *src;                    /* host [num_edges] */
    const uint32_t *dst;                    /* host [num_edges] */
    const uint16_t *label;                  /* host [num_edges], < num_labels */
    uint32_t num_labels;
    const char *const *label_names;         /* [num_labels] vocabulary for rpq_compile */
    const uint16_t *vertex_label;           /* host [num_vertices] or NULL (CRPQ condition (1)) */
    uint32_t num_vertex_labels;
    const char *const *vertex_label_names;  /* [num_vertex_labels] or NULL */
    int device;                             /* CUDA device ordinal */
    uint32_t flags;                         /* 0 or RPQ_GRAPH_IN_EDGES */
    void *cuda_stream;                      /* cudaStream_t used for the build, NULL = default */
} rpq_graph_desc;

/* Also build the per-label in-edge CSR (the transposed graph).  LGF keeps
 * in-edge slices for reverse traversal; here they serve
 * rpq_eval_targets and CRPQ atoms whose target side is bound (WavePlan's
 * reverse plans).  Doubles the graph's device memory. */
#define RPQ_GRAPH_IN_EDGES 1u

/* Copies the host arrays to the device and builds the per-label CSR.
 * Errors: EINVAL (id >= num_vertices, label >= num_labels, NULL arrays with
 * num_edges > 0), ENOMEM, ECUDA (no device).  One-time; not part of query
 * time (the paper excludes loading). */
rpq_status rpq_graph_load(const rpq_graph_desc *desc, rpq_graph **out);
void rpq_graph_free(rpq_graph *g);
/* |V|, number of DISTINCT (u,l,w) triples, number of labels */
/* Add an edge label whose edges are the given (src[i], dst[i]) pairs (device
 * arrays if on_device, else host; duplicates collapse, reading R4), with its
 * CSR (and in-edge CSR when the graph keeps in-edges).  The new label gets
 * the next id (*label_id) and can be named in regexes compiled afterwards;
 * automata compiled before stay valid (their vocabulary is a prefix).
 * Used by the loop-cache plan (rpq_cache_closure).  Mutates g: not
 * concurrently with evaluations on g.  EINVAL: bad argument, duplicate name,
 * id >= |V|; EUNSUPPORTED: >= 2^32 pairs or 65535 labels. */
rpq_status rpq_graph_add_label(rpq_graph *g, const char *name, const uint32_t *src, const uint32_t *dst,
                               uint64_t n, int on_device, void *cuda_stream, uint32_t *label_id);
rpq_status rpq_graph_info(const rpq_graph *g, uint32_t *num_vertices, uint64_t *num_edges,
                          uint32_t *num_labels);
/* Device views (valid until rpq_graph_free) of label l's CSR. */
rpq_status rpq_graph_label_csr(const rpq_graph *g, uint32_t label, const uint32_t **off,
                               const uint32_t **nbr, uint64_t *num_edges);

/* ------------------------------------------------------------------------
 * rpq_compile: regex over edge labels -> automaton (the "automata plan" of
 * P:253-259; Fig. 2(a) gives abc* as q0 -a-> q1 -b-> q2 with a c-loop).
 * Host-side.  Route: tokenise (longest match against the vocabulary, R3) ->
 * parse ('|' alternation, postfix * + ?, R2) -> Glushkov position NFA ->
 * subset construction -> Hopcroft minimisation -> trim (dead and unreachable
 * states removed) -> canonical numbering (BFS from the initial state 0).
 * If the minimal DFA has more than RPQ_MAX_STATES states the trimmed
 * Glushkov NFA is used instead (same result set, different PE).
 * flags: RPQ_SYNTAX_PAPER -> infix '+' is alternation (tab:queries,
 * P:1042-1043); RPQ_NO_MINIMIZE -> keep the Glushkov NFA (tests).
 * Errors: ESYNTAX (*err_offset = byte offset), ELABEL (*err_offset = offset
 * of the unknown name), EUNSUPPORTED (> RPQ_MAX_STATES states). */
#define RPQ_SYNTAX_PAPER 1u
#define RPQ_NO_MINIMIZE 2u
#define RPQ_MAX_STATES 64
#define RPQ_MAX_TRANSITIONS 256
#define RPQ_MAX_QUERY_LABELS 32
rpq_status rpq_compile(const rpq_graph *vocab, const char *regex, uint32_t flags,
                       rpq_nfa **out, size_t *err_offset);
/* Same, with an explicit vocabulary (no graph, no GPU needed). */
rpq_status rpq_compile_labels(const char *const *label_names, uint32_t num_labels,
                              const char *regex, uint32_t flags, rpq_nfa **out,
                              size_t *err_offset);
void rpq_nfa_free(rpq_nfa *a);
rpq_status rpq_nfa_info(const rpq_nfa *a, uint32_t *num_states, uint32_t *num_transitions,
                        uint32_t *num_final, int *accepts_empty, int *is_dfa);
/* transitions (from, label, to) sorted by (from, label, to); *n = count
 * (ECAPACITY if cap < count); final states as a bit mask */
rpq_status rpq_nfa_transitions(const rpq_nfa *a, uint32_t *from, uint32_t *label, uint32_t *to,
                               uint32_t cap, uint32_t *n, uint64_t *final_mask);
/* word membership (host simulation; used to pin the compiler) */
rpq_status rpq_nfa_accepts(const rpq_nfa *a, const uint32_t *word, uint32_t len, int *accepted);
/* Automaton of the reversed language L(rho)^R = { w_k ... w_1 : w_1 ... w_k
 * in L(rho) } (reverse every transition, the old finals become initial, the
 * old initial state final), then subset construction, minimisation, trim and
 * canonical numbering as in rpq_compile.  (x, y) in R(rho) on G  <=>
 * (y, x) in R(rho^R) on the transposed graph: the basis of single-target
 * evaluation ("single-source" mirrored; reverse plans P:867).
 * Host-side.  Errors: EINVAL (NULL), EUNSUPPORTED (> RPQ_MAX_STATES). */
rpq_status rpq_nfa_reverse(const rpq_nfa *a, rpq_nfa **out);

/* ------------------------------------------------------------------------
 * Evaluation (Definition 1): R(rho) = distinct (x, y) such that a
 * path x -> ... -> y has a label word in L(rho).  epsilon in L(rho) => (v, v)
 * for every source v (reading R1).  Method: level-synchronous multi-source
 * BFS over the product graph G x A(rho) with a per-source
 * visited set over (vertex, state) kept as bit-parallel words: source batches
 * of B sources, one bit per source, B sized against the HBM budget
 * (Challenge 2).
 * ------------------------------------------------------------------------ */
#define RPQ_COUNT 1u          /* total number of result pairs (the paper's output) */
#define RPQ_PAIRS 2u          /* materialise sorted distinct (src, dst) pairs */
#define RPQ_PER_SOURCE 4u     /* per-source result counts */
#define RPQ_STATS 8u          /* count PE / word ops / items (small overhead) */
#define RPQ_TIME_KERNELS 16u  /* CUDA-event time of every expand launch */
#define RPQ_PE 32u            /* product_edges (PE, reading R12) from the post-pass only (no in-kernel
                                 counters); in COUNT mode fused into the count pass */
#define RPQ_SOURCE_PE 64u     /* with RPQ_PER_SOURCE: per-source PE (rpq_result_source_pe); the
                                 per-source list then holds every source with a non-zero count OR PE */
#define RPQ_WCOJ 256u         /* crpq_eval: worst-case-optimal (generic) join instead of binary joins
                                 (the WCOJ-based CQ method): variables are bound one at a time and
                                 each new variable's candidates are the intersection of the sorted value
                                 lists of every atom into it; same tuples, sorted the same way */
#define RPQ_BOUNDED 128u      /* length-bounded RPQ: only paths of <= opts.max_hops edges (P:1574-1575,
                                 "length constraints ... enforced by controlling traversal depth").  Exact
                                 BFS levels: discoveries go to a separate per-level array (24 instead of 16
                                 bytes per state word, so B shrinks by 1/3); dense engine only; PE counts the
                                 out-edges of the product vertices at depth < max_hops (those expanded) */

typedef struct {
    uint32_t mode;              /* OR of the RPQ_* mode bits above; 0 = RPQ_COUNT */
    uint32_t batch_sources;     /* B; 0 = auto (HBM budget), rounded up to 64 */
    uint64_t hbm_budget_bytes;  /* 0 = 90% of free device memory */
    uint32_t shard_index;       /* evaluate batches b with b % shard_count == shard_index */
    uint32_t shard_count;       /* 0 or 1 = unsharded */
    void *cuda_stream;          /* cudaStream_t; NULL = default stream */
    uint32_t chunk_words;       /* 0 = auto; else words per work item (1,2,4,8,16,32) */
    uint32_t reserved;
    uint32_t max_hops;          /* with RPQ_BOUNDED: the length bound k >= 0 (0 = epsilon pairs only) */
    uint32_t pad0;
} rpq_eval_opts;

/* All-pairs: x ranges over all of V (R11).  With shard_count > 1 the result
 * holds only this shard's batches (sources are cut into batches of B
 * consecutive productive sources; batch b belongs to shard b % count).
 * Every rank must derive the same batches, so shard_count > 1 requires
 * batch_sources or hbm_budget_bytes (EINVAL otherwise); with an explicit
 * budget the automatic B is also capped at ceil(|P| / shard_count) rounded
 * up to 64 so that every shard gets work. */
rpq_status rpq_eval_allpairs(const rpq_graph *g, const rpq_nfa *a, const rpq_eval_opts *opts,
                             rpq_result **out);
/* The batch plan rpq_eval_allpairs would use with these options, without
 * evaluating anything (device work: the productive-source scan of
 * Challenge 2's batching): |P|, the batch width B (auto unless
 * opts->batch_sources is set), the number of batches, the 64-bit words per
 * state array and the chunk width.  Ranks of a sharded evaluation call it,
 * agree on the minimum B (all-reduce MIN) and pass it as batch_sources.
 * Errors as rpq_eval_allpairs; EINVAL for NULL arguments. */
typedef struct {
    uint64_t productive_sources;
    uint32_t batch_sources;
    uint32_t chunk_words;
    uint64_t num_batches;
    uint64_t state_words;
} rpq_plan_info;
rpq_status rpq_plan(const rpq_graph *g, const rpq_nfa *a, const rpq_eval_opts *opts, rpq_plan_info *info);

/* Loop-cache plan (WavePlan A2): evaluate `inner` over all of
 * V (PAIRS) and install R(inner) as the derived label `name`
 * (rpq_graph_add_label).  A query a (b c)* d then runs as "a name? d" with
 * inner = (b c)+: the closure is traversed once, not once per source batch.
 * opts: stream / budget / RPQ_BOUNDED as for rpq_eval_allpairs.  Errors as
 * rpq_eval_allpairs and rpq_graph_add_label. */
rpq_status rpq_cache_closure(rpq_graph *g, const rpq_nfa *inner, const char *name, const rpq_eval_opts *opts,
                             uint32_t *label_id);

/* The loop-cache plan end to end: all-pairs R(prefix (loop)* suffix) as
 * rpq_cache_closure((loop)+) into a fresh label L ("__loopN"), then
 * rpq_eval_allpairs("(prefix) L? (suffix)") with opts.  prefix / suffix may
 * be NULL or blank.  Same pairs as evaluating the regex directly (PE counts
 * the rewritten query).  Adds a label to g (see rpq_graph_add_label). */
rpq_status rpq_eval_loop_cached(rpq_graph *g, const char *prefix, const char *loop, const char *suffix,
                                const rpq_eval_opts *opts, rpq_result **out);

/* Single source x = src.  src >= |V| -> EINVAL. */
rpq_status rpq_eval_single_source(const rpq_graph *g, const rpq_nfa *a, uint32_t src,
                                  const rpq_eval_opts *opts, rpq_result **out);
/* A set of sources (host array, any order, no duplicates -> else EINVAL).
 * Pairs are sorted by (src, dst) regardless of input order. */
rpq_status rpq_eval_sources(const rpq_graph *g, const rpq_nfa *a, const uint32_t *srcs,
                            uint64_t n, const rpq_eval_opts *opts, rpq_result **out);
/* A set of TARGETS (host array, any order, no duplicates -> else EINVAL):
 * the pairs (x, t) of R(rho) with t in targets and x in V, evaluated
 * backwards -- rpq_nfa_reverse(a) traversed over the in-edge CSR from the
 * targets (the graph must have been loaded with RPQ_GRAPH_IN_EDGES, else
 * EUNSUPPORTED).  Result columns are (x, t) as for the forward calls, but
 * rows are sorted by (t, x) (grouped by target); RPQ_PER_SOURCE gives
 * per-TARGET counts.  epsilon in L(rho) => (t, t) for every target. */
rpq_status rpq_eval_targets(const rpq_graph *g, const rpq_nfa *a, const uint32_t *targets,
                            uint64_t n, const rpq_eval_opts *opts, rpq_result **out);
/* Single target t: { (x, t) }, sorted by x.  t >= |V| -> EINVAL. */
rpq_status rpq_eval_single_target(const rpq_graph *g, const rpq_nfa *a, uint32_t t,
                                  const rpq_eval_opts *opts, rpq_result **out);

/* Output beyond HBM (the paper's outputs reach 2.4 T pairs
 * and are materialised through host memory): the
 * all-pairs result delivered to the host in (src, dst) order through `sink`,
 * in pieces of at most piece_pairs pairs (0 = 2^26); the host pointers are
 * valid during the call only.  A PER_SOURCE pass sizes the output; sources
 * are then evaluated in chunks of consecutive vertex ids whose pairs fit
 * device_budget_bytes (0 = a quarter of the free device memory; a single
 * source always forms a chunk), each chunk in PAIRS mode, and its pairs are
 * copied through two pinned host buffers so that the copy of piece k+1
 * overlaps the sink of piece k.  Sharding: chunk c belongs to shard
 * c % shard_count; the chunks follow device_budget_bytes, so a sharded call
 * must pass the same non-zero budget on every rank (EINVAL if 0).  *total = pairs delivered.  A sink returning non-zero
 * stops the evaluation early (RPQ_OK; *total counts what was delivered).
 * Errors as rpq_eval_allpairs; EINVAL for a NULL sink. */
typedef int (*rpq_pairs_sink)(const uint32_t *src, const uint32_t *dst, uint64_t n, void *ctx);
rpq_status rpq_eval_allpairs_stream(const rpq_graph *g, const rpq_nfa *a, const rpq_eval_opts *opts,
                                    uint64_t device_budget_bytes, uint64_t piece_pairs,
                                    rpq_pairs_sink sink, void *ctx, uint64_t *total);

/* ------------------------------------------------------------------------
 * CRPQ (Definition 2): all homomorphisms f: V_q -> V with
 * (1) L(f(u)) = L_q(u) where a label is given, (2) (f(x), f(y)) in R(rho) for
 * every atom x -rho-> y; plus optional distinct-vertex filters (CQ4/CQ5,
 * P:1085).  Atoms are evaluated with the RPQ kernels (sources restricted to
 * candidates), then joined on the device.  Tuples are distinct and sorted
 * lexicographically in variable order.  A variable in no atom or a
 * disconnected pattern -> EUNSUPPORTED (reading R18).
 * ------------------------------------------------------------------------ */
typedef struct {
    uint32_t num_vars;
    const int32_t *var_label;        /* [num_vars] vertex-label id or -1 (any) */
    const int64_t *var_const;        /* [num_vars] vertex id or -1 (free) */
    uint32_t num_atoms;
    const uint32_t *atom_x;          /* [num_atoms] variable ids */
    const uint32_t *atom_y;
    const rpq_nfa *const *atom_nfa;  /* [num_atoms] */
    uint32_t num_distinct;
    const uint32_t *distinct_pairs;  /* [2*num_distinct] variable ids */
} crpq_query;
rpq_status crpq_eval(const rpq_graph *g, const crpq_query *q, const rpq_eval_opts *opts,
                     rpq_result **out);
/* crpq_eval projected onto out_vars (distinct variable ids, in that column
 * order): the distinct tuples of those variables over all homomorphisms,
 * sorted lexicographically.  EINVAL for an empty / repeated / out-of-range
 * list. */
rpq_status crpq_eval_project(const rpq_graph *g, const crpq_query *q, const uint32_t *out_vars, uint32_t num_out,
                             const rpq_eval_opts *opts, rpq_result **out);
/* Start-in-the-middle plan (WavePlan A3/A4) for
 * R(alpha mid beta): exploration starts at the edges of the middle
 * expression `mid` (typically one selective label) -- alpha is traversed
 * backwards (reversed automaton, in-edge CSR when loaded: "with transpose")
 * and beta forwards -- and the distinct (x, y) pairs are enumerated, sorted
 * and deduplicated (they cannot be produced in source order).  Runs as the
 * CRPQ x -alpha-> u -mid-> w -beta-> y (RPQ_WCOJ, matching order from the
 * middle) projected on (x, y).  Same pairs as rpq_eval_allpairs on
 * "(alpha)(mid)(beta)".  Errors as rpq_compile / crpq_eval. */
rpq_status rpq_eval_middle(const rpq_graph *g, const char *alpha, const char *mid, const char *beta,
                           const rpq_eval_opts *opts, rpq_result **out);

/* ------------------------------------------------------------------------
 * Results.  Pair results have 2 columns (src, dst); CRPQ results one column
 * per variable.  Rows are distinct and sorted.  Device views stay valid
 * until rpq_result_free.
 * ------------------------------------------------------------------------ */
#define RPQ_MAX_COLS 16
typedef struct {
    uint64_t count;             /* result pairs / tuples */
    uint64_t product_edges;     /* PE: sum over reached (v,q) of product out-degree (RPQ_STATS) */
    uint64_t word_items;        /* non-zero 64-bit frontier words expanded */
    uint64_t word_edge_ops;     /* (non-zero frontier word) x (edge) operations */
    uint64_t items;             /* work items (chunk of words, state, vertex) expanded */
    uint64_t item_edges;        /* (item) x (edge) pairs = neighbour ids read */
    uint64_t item_transitions;  /* (item) x (automaton transition) pairs = offset pairs read */
    uint64_t activations;       /* red.or on the activity bitmap (row, chunk) */
    uint64_t next_reds;         /* red.or on the next-frontier words */
    uint32_t levels;            /* BFS levels summed over batches */
    uint32_t batches;           /* batches evaluated by this shard */
    uint32_t batch_sources;     /* B */
    uint32_t chunk_words;       /* words per work item */
    uint64_t productive_sources;/* |P| over the whole query (all shards) */
    uint64_t state_words;       /* 64-bit words per state array */
    uint64_t expand_launches;   /* expand-kernel launches (main + hub) */
    uint64_t kernel_launches;   /* all kernels this library launched for the call */
    double expand_ms;           /* RPQ_TIME_KERNELS: summed CUDA-event time of expand launches */
    double total_ms;            /* CUDA-event time from entry to result ready */
    uint64_t pull_levels;       /* levels run bottom-up (direction-optimising), over batches */
    uint64_t pull_loads;        /* in-neighbour visited-word loads of the pull levels */
    uint64_t pull_words;        /* (row, word) pairs scanned by the pull levels */
    uint64_t adv_words;         /* words read by the top-down advance (Vis + Done of active chunks) */
    uint64_t adv_zero_sectors;  /* ... 4-word sectors of those without frontier bits */
} rpq_stats;

uint64_t rpq_result_count(const rpq_result *r);
rpq_status rpq_result_device_view(const rpq_result *r, const uint32_t **cols, uint32_t *ncols,
                                  uint64_t *n);
/* copies rows to host column buffers cols[0..ncols-1] of capacity cap rows;
 * ECAPACITY (and *n = required) if cap < rows */
rpq_status rpq_result_copy_host(const rpq_result *r, uint32_t *const *cols, uint64_t cap,
                                uint64_t *n);
/* RPQ_PER_SOURCE: (source, count) for every source of this shard with a
 * non-zero count, ascending source; host buffers, ECAPACITY as above */
rpq_status rpq_result_source_counts(const rpq_result *r, uint32_t *srcs, uint64_t *counts,
                                    uint64_t cap, uint64_t *n);
/* RPQ_PER_SOURCE | RPQ_SOURCE_PE: product edges traversed per listed source
 * (same order as rpq_result_source_counts): sum over the (vertex, state)
 * pairs the source reaches of the product out-degree on the minimal trim DFA
 * (reading R12).  Host buffer; ECAPACITY as above; EINVAL if
 * the result has no per-source PE. */
rpq_status rpq_result_source_pe(const rpq_result *r, uint64_t *pe, uint64_t cap, uint64_t *n);
rpq_status rpq_result_stats(const rpq_result *r, rpq_stats *s);
/* PAIRS results of rpq_eval_allpairs / rpq_eval_sources (and PER_SOURCE
 * results of the dense engine; other results: no entries): the batches this
 * shard evaluated, in order.  Batch k covers the candidate
 * sources [cand_lo, cand_hi) (indices into the sorted candidate list; the
 * vertex ids themselves for all-pairs) and owns result rows [offset,
 * offset + count); batches of all shards, sorted by cand_lo, tile the
 * global (src, dst)-sorted result -- which is how a multi-GPU gather places
 * every shard's rows.  Host buffer of capacity
 * cap entries; *n = entries (ECAPACITY if cap < *n; 0 for other modes). */
typedef struct {
    uint64_t cand_lo, cand_hi;
    uint64_t offset, count;
} rpq_batch_info;
rpq_status rpq_result_batches(const rpq_result *r, rpq_batch_info *out, uint64_t cap, uint64_t *n);
void rpq_result_free(rpq_result *r);

/* Host-only: the shard that owns each candidate source under the batch plan
 * of rpq_eval_* (productive candidates pidx[0..np) ascending, batches of
 * batch_sources consecutive productive sources, batch b -> shard
 * b % shard_count; non-productive candidates belong to the batch before them,
 * and all to shard 0 when np == 0).  owner: host [nsrc].  Used to test and
 * reason about multi-GPU sharding without a GPU. */
rpq_status rpq_shard_plan(const uint32_t *pidx, uint64_t np, uint64_t nsrc, uint64_t batch_sources,
                          uint32_t shard_count, uint32_t *owner);

const char *rpq_last_error(void);
/* number of usable CUDA devices (0 on a machine without a GPU) */
rpq_status rpq_device_count(int *n);
/* library build string (arch, version) */
const char *rpq_version(void);
/* Device memory: per-batch state arrays and result buffers (pairs, CRPQ
 * tuples, per-source counts) come from the device's stream-ordered memory
 * pool, which keeps freed blocks reserved so that repeated evaluations do not
 * pay for page mapping (cudaMalloc of a 64 GB pair buffer took 26 ms on a
 * B200).  rpq_trim_memory returns the reserved but unused bytes of `device`'s
 * pool to the driver (e.g. before handing HBM to another allocator).
 * RPQ_EINVAL if device is not a CUDA device; RPQ_ECUDA on driver errors. */
rpq_status rpq_trim_memory(int device);
/* Replace the pool by the caller's device allocator (e.g. a framework's
 * caching allocator): alloc(bytes, stream, ctx) returns device memory usable
 * in stream order on `stream` (NULL on failure -> RPQ_ENOMEM), free_(ptr,
 * stream, ctx) releases it.  Both NULL restores the pool.  Set it before any
 * graph/evaluation whose buffers it should hold: graphs and results free
 * their buffers through the allocator that was installed when they were
 * created (so the functions must stay valid until then), results on the
 * stream of the evaluation that made them (that stream must outlive the
 * result).  Process-wide.
 * EINVAL if exactly one of the two functions is NULL. */
rpq_status rpq_set_allocator(void *(*alloc)(size_t bytes, void *stream, void *ctx),
                             void (*free_)(void *ptr, void *stream, void *ctx), void *ctx);

#ifdef __cplusplus
}
#endif
#endif /* RPQ_H */
