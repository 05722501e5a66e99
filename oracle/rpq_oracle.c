/*
 * oracle/rpq_oracle.c -- O1, the primary CPU oracle for RPQ evaluation.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA product path in
 * paper_2602_20748_b200/ (and includes nothing from it).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   Definition 1: the set of DISTINCT pairs (x, y) such that some
 *   path x -> ... -> y has an edge-label word in L(rho).  It follows the
 *   automata-based approach of P:252-257 step by step: for each starting
 *   vertex, traverse the product graph G x A(rho) from (x, q_init), keep a
 *   per-source visited set over (vertex, automaton-state) pairs, and emit
 *   (x, y) whenever a final state is reached at vertex y.  Traversal order is
 *   breadth-first (a plain FIFO queue); any complete traversal reaches the
 *   same set.
 *
 * Two automata are built from the regex, by textbook constructions written
 * out below (not the product's Glushkov/Hopcroft route):
 *   - a Thompson epsilon-NFA (used by og_eval(..., use_dfa=0));
 *   - its subset-construction DFA, completed, Moore-minimised and trimmed
 *     (used by og_eval(..., use_dfa=1); it defines the product-edge count PE
 *     of SURVEY.md §8(d) / DESIGN.md reading R12).
 * Both modes must give identical pair sets (tests check this).
 *
 * Readings:
 *   R1  epsilon in L(rho) => (v, v) is a result for every v.
 *   R2  default dialect: '|' alternation, postfix '*' '+' '?'; paper dialect
 *       (tab:queries): infix '+' is alternation.
 *   R3  labels are tokenised by longest match against the vocabulary;
 *       whitespace, '.' and '/' are optional explicit concatenation.
 *   R4  E is a SET of (u, label, w) triples (duplicates collapse).
 *   R5  self-loops are 1-hop paths.
 *
 * Length bound (og_eval_bounded; "length constraints can be
 * naturally enforced by controlling traversal depth"): the same BFS, but a
 * product vertex first reached at depth d is expanded only if d < max_hops,
 * so (x, y) is emitted iff some path of length <= max_hops has a word in
 * L(rho); PE then counts the out-edges of the expanded vertices only.
 *
 * Parity pins: see tests/test_oracle.py (paper's worked example P:84, P:104,
 * P:236; brute-force Definition 1; relational algebra; closed forms).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <pthread.h>

#define OG_OK 0
#define OG_ESYNTAX (-2)
#define OG_ELABEL (-3)
#define OG_ENOMEM (-4)
#define OG_EINVAL (-1)

/* ======================================================================
 * Graph: G = (V, E, L) of P:182-183, edges as distinct (u, l, w) triples.
 * Adjacency adj[off[l*nv+u] .. off[l*nv+u+1]) = sorted distinct w with
 * (u, l, w) in E.
 * ====================================================================== */
typedef struct {
    uint32_t nv, nl;
    uint64_t ne;
    uint64_t *off;
    uint32_t *adj;
} og_graph;

static int cmp_u32(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

og_graph *og_graph_new(uint32_t nv, uint64_t ne, const uint32_t *src,
                       const uint32_t *dst, const uint16_t *lab, uint32_t nl) {
    og_graph *g = (og_graph *)calloc(1, sizeof(og_graph));
    if (!g) return NULL;
    g->nv = nv; g->nl = nl;
    uint64_t nslots = (uint64_t)nl * nv;
    g->off = (uint64_t *)calloc(nslots + 1, sizeof(uint64_t));
    uint32_t *tmp = (uint32_t *)malloc((ne ? ne : 1) * sizeof(uint32_t));
    if (!g->off || !tmp) { free(g->off); free(tmp); free(g); return NULL; }
    for (uint64_t i = 0; i < ne; i++) {
        if (src[i] >= nv || dst[i] >= nv || lab[i] >= nl) {
            free(g->off); free(tmp); free(g); return NULL;
        }
        g->off[(uint64_t)lab[i] * nv + src[i] + 1]++;
    }
    for (uint64_t s = 0; s < nslots; s++) g->off[s + 1] += g->off[s];
    uint64_t *fill = (uint64_t *)malloc((nslots ? nslots : 1) * sizeof(uint64_t));
    if (!fill) { free(g->off); free(tmp); free(g); return NULL; }
    memcpy(fill, g->off, nslots * sizeof(uint64_t));
    for (uint64_t i = 0; i < ne; i++)
        tmp[fill[(uint64_t)lab[i] * nv + src[i]]++] = dst[i];
    free(fill);
    /* sort each list and drop duplicate triples (reading R4) */
    uint64_t outpos = 0;
    uint64_t start = 0;
    for (uint64_t s = 0; s < nslots; s++) {
        uint64_t end = g->off[s + 1];
        uint64_t n = end - start;
        if (n > 1) qsort(tmp + start, n, sizeof(uint32_t), cmp_u32);
        uint64_t new_start = outpos;
        for (uint64_t k = start; k < end; k++) {
            if (k > start && tmp[k] == tmp[k - 1]) continue;
            tmp[outpos++] = tmp[k];
        }
        g->off[s] = new_start;
        start = end;
    }
    g->off[nslots] = outpos;
    g->ne = outpos;
    g->adj = tmp;
    return g;
}

void og_graph_free(og_graph *g) {
    if (!g) return;
    free(g->off); free(g->adj); free(g);
}

uint64_t og_graph_num_edges(const og_graph *g) { return g->ne; }

static inline uint64_t deg(const og_graph *g, uint32_t l, uint32_t u) {
    uint64_t s = (uint64_t)l * g->nv + u;
    return g->off[s + 1] - g->off[s];
}

/* ======================================================================
 * Regex AST and parser (grammar of tab:queries P:1039-1043 and readings
 * R2/R3).  alt := concat ('|' concat)* ; concat := postfix+ ;
 * postfix := atom ('*' | '+' | '?')* ; atom := LABEL | '(' alt ')'.
 * ====================================================================== */
enum { N_LABEL, N_CONCAT, N_ALT, N_STAR, N_PLUS, N_OPT };
typedef struct node { int kind, label, a, b; } node;   /* a, b: child indices, -1 = none */

typedef struct {
    const char *s; size_t pos, len;
    const char *const *names; uint32_t nnames;
    int paper;             /* 1 => infix '+' is alternation */
    int err; size_t err_off;
    node *pool; int npool, cap;
} parser;

/* appends a node; returns its index or -1 (out of memory) */
static int mk(parser *p, int kind, int label, int a, int b) {
    if (p->npool == p->cap) {
        int nc = p->cap ? p->cap * 2 : 64;
        node *np_ = (node *)realloc(p->pool, nc * sizeof(node));
        if (!np_) { p->err = OG_ENOMEM; return -1; }
        p->pool = np_; p->cap = nc;
    }
    node *n = &p->pool[p->npool];
    n->kind = kind; n->label = label; n->a = a; n->b = b;
    return p->npool++;
}

static void skip_sep(parser *p) {
    while (p->pos < p->len) {
        char c = p->s[p->pos];
        if (c == ' ' || c == '\t' || c == '\n' || c == '.' || c == '/') p->pos++;
        else break;
    }
}

static int peek(parser *p) { skip_sep(p); return p->pos < p->len ? p->s[p->pos] : 0; }

static int is_op(int c) { return c == '(' || c == ')' || c == '|' || c == '*' || c == '+' || c == '?'; }

/* longest vocabulary name matching at p->pos (reading R3) */
static int match_label(parser *p, size_t *mlen) {
    int best = -1; size_t bl = 0;
    for (uint32_t i = 0; i < p->nnames; i++) {
        size_t l = strlen(p->names[i]);
        if (l == 0 || l > p->len - p->pos) continue;
        if (memcmp(p->s + p->pos, p->names[i], l) == 0 && l > bl) { best = (int)i; bl = l; }
    }
    *mlen = bl;
    return best;
}

static int parse_alt(parser *p);

static int parse_atom(parser *p) {
    int c = peek(p);
    if (c == '(') {
        p->pos++;
        int r = parse_alt(p);
        if (p->err) return -1;
        if (peek(p) != ')') { p->err = OG_ESYNTAX; p->err_off = p->pos; return -1; }
        p->pos++;
        return r;
    }
    if (c == 0 || is_op(c)) { p->err = OG_ESYNTAX; p->err_off = p->pos; return -1; }
    size_t ml;
    int lab = match_label(p, &ml);
    if (lab < 0) { p->err = OG_ELABEL; p->err_off = p->pos; return -1; }
    p->pos += ml;
    return mk(p, N_LABEL, lab, -1, -1);
}

static int parse_postfix(parser *p) {
    int r = parse_atom(p);
    if (p->err) return -1;
    for (;;) {
        int c = peek(p);
        int kind;
        if (c == '*') kind = N_STAR;
        else if (c == '?') kind = N_OPT;
        else if (c == '+' && !p->paper) kind = N_PLUS;
        else break;
        p->pos++;
        r = mk(p, kind, -1, r, -1);
        if (r < 0) return -1;
    }
    return r;
}

static int starts_atom(parser *p) {
    int c = peek(p);
    return c != 0 && (c == '(' || !is_op(c));
}

static int parse_concat(parser *p) {
    int r = parse_postfix(p);
    if (p->err) return -1;
    while (starts_atom(p)) {
        int q = parse_postfix(p);
        if (p->err) return -1;
        r = mk(p, N_CONCAT, -1, r, q);
        if (r < 0) return -1;
    }
    return r;
}

static int parse_alt(parser *p) {
    int r = parse_concat(p);
    if (p->err) return -1;
    for (;;) {
        int c = peek(p);
        if (!(c == '|' || (c == '+' && p->paper))) break;
        p->pos++;
        int q = parse_concat(p);
        if (p->err) return -1;
        r = mk(p, N_ALT, -1, r, q);
        if (r < 0) return -1;
    }
    return r;
}

/* ======================================================================
 * Thompson construction (epsilon-NFA).  label -1 = epsilon move.
 * ====================================================================== */
typedef struct { int from, to, label; } tedge;
typedef struct {
    int nstates, start, accept;
    tedge *e; int ne, cap;
} tnfa;

static int t_state(tnfa *t) { return t->nstates++; }
static int t_edge(tnfa *t, int f, int to, int l) {
    if (t->ne == t->cap) {
        int nc = t->cap ? 2 * t->cap : 64;
        tedge *ne_ = (tedge *)realloc(t->e, nc * sizeof(tedge));
        if (!ne_) return -1;
        t->e = ne_; t->cap = nc;
    }
    t->e[t->ne].from = f; t->e[t->ne].to = to; t->e[t->ne].label = l; t->ne++;
    return 0;
}

/* builds a fragment for node i; returns start/accept through s,a */
static int thompson(tnfa *t, node *pool, int i, int *s, int *a) {
    node *n = &pool[i];
    int s1, a1, s2, a2;
    int ia = n->a, ib = n->b;
    switch (n->kind) {
    case N_LABEL:
        *s = t_state(t); *a = t_state(t);
        return t_edge(t, *s, *a, n->label);
    case N_CONCAT:
        if (thompson(t, pool, ia, &s1, &a1) || thompson(t, pool, ib, &s2, &a2)) return -1;
        *s = s1; *a = a2;
        return t_edge(t, a1, s2, -1);
    case N_ALT:
        if (thompson(t, pool, ia, &s1, &a1) || thompson(t, pool, ib, &s2, &a2)) return -1;
        *s = t_state(t); *a = t_state(t);
        return t_edge(t, *s, s1, -1) | t_edge(t, *s, s2, -1) |
               t_edge(t, a1, *a, -1) | t_edge(t, a2, *a, -1);
    case N_STAR:   /* rho* : zero or more */
        if (thompson(t, pool, ia, &s1, &a1)) return -1;
        *s = t_state(t); *a = t_state(t);
        return t_edge(t, *s, s1, -1) | t_edge(t, *s, *a, -1) |
               t_edge(t, a1, s1, -1) | t_edge(t, a1, *a, -1);
    case N_PLUS:   /* rho+ : one or more */
        if (thompson(t, pool, ia, &s1, &a1)) return -1;
        *s = t_state(t); *a = t_state(t);
        return t_edge(t, *s, s1, -1) | t_edge(t, a1, s1, -1) | t_edge(t, a1, *a, -1);
    case N_OPT:    /* rho? : zero or one */
        if (thompson(t, pool, ia, &s1, &a1)) return -1;
        *s = t_state(t); *a = t_state(t);
        return t_edge(t, *s, s1, -1) | t_edge(t, *s, *a, -1) | t_edge(t, a1, *a, -1);
    }
    return -1;
}

/* ======================================================================
 * Automaton object: Thompson NFA + minimal trim DFA.
 * ====================================================================== */
typedef struct {
    /* Thompson NFA */
    int tn;                  /* states */
    int tstart, taccept;
    int *tlab_off;           /* [tn+1] labelled (non-eps) out-moves per state */
    int *tlab_label, *tlab_to;
    uint64_t *closure;       /* [tn * cw] epsilon-closure bitsets */
    int cw;                  /* words per bitset */
    int accepts_empty;
    /* minimal trim DFA: state 0 is initial */
    int dn;
    int nalpha;              /* labels used */
    int *alpha;              /* [nalpha] label ids */
    int *dnext;              /* [dn * nalpha], -1 = undefined (dead, trimmed) */
    unsigned char *dfinal;   /* [dn] */
    uint32_t nlabels_vocab;
} og_automaton;

static int bs_test(const uint64_t *b, int i) { return (int)((b[i >> 6] >> (i & 63)) & 1); }
static void bs_set(uint64_t *b, int i) { b[i >> 6] |= 1ull << (i & 63); }

static void eps_closure(const tnfa *t, int q, uint64_t *out, int *stack) {
    int sp = 0;
    bs_set(out, q); stack[sp++] = q;
    while (sp) {
        int x = stack[--sp];
        for (int k = 0; k < t->ne; k++)
            if (t->e[k].from == x && t->e[k].label < 0 && !bs_test(out, t->e[k].to)) {
                bs_set(out, t->e[k].to); stack[sp++] = t->e[k].to;
            }
    }
}

void og_automaton_free(og_automaton *A) {
    if (!A) return;
    free(A->tlab_off); free(A->tlab_label); free(A->tlab_to); free(A->closure);
    free(A->alpha); free(A->dnext); free(A->dfinal); free(A);
}

/* subset construction -> complete DFA -> Moore minimisation -> trim */
static int build_min_dfa(og_automaton *A, const tnfa *t) {
    int cw = A->cw, tn = A->tn;
    /* alphabet: labels occurring in the regex, ascending */
    int *seen = (int *)calloc(A->nlabels_vocab ? A->nlabels_vocab : 1, sizeof(int));
    if (!seen) return OG_ENOMEM;
    for (int k = 0; k < t->ne; k++) if (t->e[k].label >= 0) seen[t->e[k].label] = 1;
    A->nalpha = 0;
    A->alpha = (int *)malloc(sizeof(int) * (A->nlabels_vocab ? A->nlabels_vocab : 1));
    for (uint32_t l = 0; l < A->nlabels_vocab; l++) if (seen[l]) A->alpha[A->nalpha++] = (int)l;
    free(seen);
    int na = A->nalpha;

    /* subset construction over epsilon-closed sets; set index 0 = start */
    int cap = 16, ns = 0;
    uint64_t *sets = (uint64_t *)calloc((size_t)cap * cw, sizeof(uint64_t));
    int *trans = (int *)malloc(sizeof(int) * (size_t)cap * (na ? na : 1));
    uint64_t *tmp = (uint64_t *)calloc(cw, sizeof(uint64_t));
    memcpy(sets, A->closure + (size_t)A->tstart * cw, cw * sizeof(uint64_t));
    ns = 1;
    for (int d = 0; d < ns; d++) {
        for (int ai = 0; ai < na; ai++) {
            memset(tmp, 0, cw * sizeof(uint64_t));
            int any = 0;
            for (int q = 0; q < tn; q++) {
                if (!bs_test(sets + (size_t)d * cw, q)) continue;
                for (int k = A->tlab_off[q]; k < A->tlab_off[q + 1]; k++)
                    if (A->tlab_label[k] == A->alpha[ai]) {
                        const uint64_t *c = A->closure + (size_t)A->tlab_to[k] * cw;
                        for (int w = 0; w < cw; w++) tmp[w] |= c[w];
                        any = 1;
                    }
            }
            int target = -1;
            if (any) {
                for (int e = 0; e < ns; e++)
                    if (!memcmp(sets + (size_t)e * cw, tmp, cw * sizeof(uint64_t))) { target = e; break; }
                if (target < 0) {
                    if (ns == cap) {
                        cap *= 2;
                        sets = (uint64_t *)realloc(sets, (size_t)cap * cw * sizeof(uint64_t));
                        trans = (int *)realloc(trans, sizeof(int) * (size_t)cap * (na ? na : 1));
                    }
                    memcpy(sets + (size_t)ns * cw, tmp, cw * sizeof(uint64_t));
                    target = ns++;
                }
            }
            trans[(size_t)d * na + ai] = target;
        }
    }
    /* complete the DFA with an explicit dead state `ns` */
    int N = ns + 1, dead = ns;
    int *delta = (int *)malloc(sizeof(int) * (size_t)N * (na ? na : 1));
    int *fin = (int *)calloc(N, sizeof(int));
    for (int d = 0; d < ns; d++) {
        fin[d] = bs_test(sets + (size_t)d * cw, A->taccept);
        for (int ai = 0; ai < na; ai++) {
            int x = trans[(size_t)d * na + ai];
            delta[(size_t)d * na + ai] = x < 0 ? dead : x;
        }
    }
    for (int ai = 0; ai < na; ai++) delta[(size_t)dead * na + ai] = dead;
    free(sets); free(trans); free(tmp);

    /* Moore: refine {final, non-final} by transition signatures to a fixpoint */
    int *cls = (int *)malloc(sizeof(int) * N), *ncls = (int *)malloc(sizeof(int) * N);
    int *sig = (int *)malloc(sizeof(int) * (size_t)N * (na + 1));
    int ncl = 0;
    for (int d = 0; d < N; d++) cls[d] = fin[d];
    for (int d = 0; d < N; d++) if (cls[d] + 1 > ncl) ncl = cls[d] + 1;
    for (;;) {
        for (int d = 0; d < N; d++) {
            sig[(size_t)d * (na + 1)] = cls[d];
            for (int ai = 0; ai < na; ai++) sig[(size_t)d * (na + 1) + 1 + ai] = cls[delta[(size_t)d * na + ai]];
        }
        int nn = 0;
        for (int d = 0; d < N; d++) {
            ncls[d] = -1;
            for (int e = 0; e < d; e++)
                if (!memcmp(sig + (size_t)e * (na + 1), sig + (size_t)d * (na + 1), sizeof(int) * (na + 1))) {
                    ncls[d] = ncls[e]; break;
                }
            if (ncls[d] < 0) ncls[d] = nn++;
        }
        int stable = (nn == ncl);
        memcpy(cls, ncls, sizeof(int) * N);
        ncl = nn;
        if (stable) break;
    }
    /* quotient automaton over classes */
    int *qd = (int *)malloc(sizeof(int) * (size_t)ncl * (na ? na : 1));
    int *qf = (int *)calloc(ncl, sizeof(int));
    for (int d = 0; d < N; d++) {
        qf[cls[d]] = fin[d];
        for (int ai = 0; ai < na; ai++) qd[(size_t)cls[d] * na + ai] = cls[delta[(size_t)d * na + ai]];
    }
    /* trim: keep classes reachable from start AND co-reachable to a final */
    int *reach = (int *)calloc(ncl, sizeof(int)), *coreach = (int *)calloc(ncl, sizeof(int));
    int *stack = (int *)malloc(sizeof(int) * (ncl + 1));
    int sp = 0;
    reach[cls[0]] = 1; stack[sp++] = cls[0];
    while (sp) {
        int x = stack[--sp];
        for (int ai = 0; ai < na; ai++) { int y = qd[(size_t)x * na + ai]; if (!reach[y]) { reach[y] = 1; stack[sp++] = y; } }
    }
    for (int c = 0; c < ncl; c++) coreach[c] = qf[c];
    for (int changed = 1; changed;) {
        changed = 0;
        for (int c = 0; c < ncl; c++) if (!coreach[c])
            for (int ai = 0; ai < na; ai++) if (coreach[qd[(size_t)c * na + ai]]) { coreach[c] = 1; changed = 1; break; }
    }
    /* canonical renumbering: BFS from the start class, labels ascending */
    int *newid = (int *)malloc(sizeof(int) * ncl);
    for (int c = 0; c < ncl; c++) newid[c] = -1;
    int *order = (int *)malloc(sizeof(int) * ncl);
    int no = 0, head = 0;
    if (reach[cls[0]] && coreach[cls[0]]) { newid[cls[0]] = no; order[no++] = cls[0]; }
    while (head < no) {
        int x = order[head++];
        for (int ai = 0; ai < na; ai++) {
            int y = qd[(size_t)x * na + ai];
            if (reach[y] && coreach[y] && newid[y] < 0) { newid[y] = no; order[no++] = y; }
        }
    }
    A->dn = no;
    A->dnext = (int *)malloc(sizeof(int) * (size_t)(no ? no : 1) * (na ? na : 1));
    A->dfinal = (unsigned char *)calloc(no ? no : 1, 1);
    for (int i = 0; i < no; i++) {
        int x = order[i];
        A->dfinal[i] = (unsigned char)qf[x];
        for (int ai = 0; ai < na; ai++) {
            int y = qd[(size_t)x * na + ai];
            A->dnext[(size_t)i * na + ai] = newid[y];   /* -1 if trimmed */
        }
    }
    free(delta); free(fin); free(cls); free(ncls); free(sig); free(qd); free(qf);
    free(reach); free(coreach); free(stack); free(newid); free(order);
    return OG_OK;
}

og_automaton *og_compile(const char *regex, const char *const *names, uint32_t nnames,
                         int paper_dialect, int *status, size_t *err_off) {
    parser p; memset(&p, 0, sizeof(p));
    p.s = regex; p.len = strlen(regex); p.names = names; p.nnames = nnames; p.paper = paper_dialect;
    *status = OG_OK; if (err_off) *err_off = 0;
    int root = parse_alt(&p);
    if (!p.err && peek(&p) != 0) { p.err = OG_ESYNTAX; p.err_off = p.pos; }
    if (p.err) { *status = p.err; if (err_off) *err_off = p.err_off; free(p.pool); return NULL; }
    tnfa t; memset(&t, 0, sizeof(t));
    int s, a;
    if (thompson(&t, p.pool, root, &s, &a)) { free(p.pool); free(t.e); *status = OG_ENOMEM; return NULL; }
    free(p.pool);
    og_automaton *A = (og_automaton *)calloc(1, sizeof(og_automaton));
    A->nlabels_vocab = nnames;
    A->tn = t.nstates; A->tstart = s; A->taccept = a;
    A->cw = (A->tn + 63) / 64;
    /* labelled moves grouped by source state */
    A->tlab_off = (int *)calloc(A->tn + 1, sizeof(int));
    int nl = 0;
    for (int k = 0; k < t.ne; k++) if (t.e[k].label >= 0) { A->tlab_off[t.e[k].from + 1]++; nl++; }
    for (int q = 0; q < A->tn; q++) A->tlab_off[q + 1] += A->tlab_off[q];
    A->tlab_label = (int *)malloc(sizeof(int) * (nl ? nl : 1));
    A->tlab_to = (int *)malloc(sizeof(int) * (nl ? nl : 1));
    int *fillp = (int *)malloc(sizeof(int) * (A->tn + 1));
    memcpy(fillp, A->tlab_off, sizeof(int) * (A->tn + 1));
    for (int k = 0; k < t.ne; k++) if (t.e[k].label >= 0) {
        int pos = fillp[t.e[k].from]++;
        A->tlab_label[pos] = t.e[k].label; A->tlab_to[pos] = t.e[k].to;
    }
    free(fillp);
    /* epsilon closures */
    A->closure = (uint64_t *)calloc((size_t)A->tn * A->cw, sizeof(uint64_t));
    int *stack = (int *)malloc(sizeof(int) * (A->tn + 1) * 4);
    for (int q = 0; q < A->tn; q++) eps_closure(&t, q, A->closure + (size_t)q * A->cw, stack);
    free(stack);
    A->accepts_empty = bs_test(A->closure + (size_t)A->tstart * A->cw, A->taccept);
    int st = build_min_dfa(A, &t);
    free(t.e);
    if (st) { og_automaton_free(A); *status = st; return NULL; }
    return A;
}

/* info: which=0 Thompson NFA, which=1 minimal trim DFA */
void og_automaton_info(const og_automaton *A, int which, int *nstates, int *ntrans,
                       int *accepts_empty, int *nfinal) {
    if (which == 0) {
        *nstates = A->tn; *ntrans = A->tlab_off[A->tn]; *nfinal = 1;
    } else {
        int nt = 0, nf = 0;
        for (int d = 0; d < A->dn; d++) {
            nf += A->dfinal[d];
            for (int ai = 0; ai < A->nalpha; ai++) nt += A->dnext[(size_t)d * A->nalpha + ai] >= 0;
        }
        *nstates = A->dn; *ntrans = nt; *nfinal = nf;
    }
    *accepts_empty = A->accepts_empty;
}

/* DFA transitions as (from, label, to) triples; returns count */
int og_dfa_transitions(const og_automaton *A, int *from, int *label, int *to, int cap) {
    int n = 0;
    for (int d = 0; d < A->dn; d++)
        for (int ai = 0; ai < A->nalpha; ai++) {
            int y = A->dnext[(size_t)d * A->nalpha + ai];
            if (y < 0) continue;
            if (n < cap) { from[n] = d; label[n] = A->alpha[ai]; to[n] = y; }
            n++;
        }
    return n;
}

int og_dfa_is_final(const og_automaton *A, int d) { return d >= 0 && d < A->dn ? A->dfinal[d] : 0; }

/* word membership, both automata (used to pin the compilers against Python re) */
int og_accepts(const og_automaton *A, int use_dfa, const int *word, int len) {
    if (use_dfa) {
        if (A->dn == 0) return 0;
        int d = 0;
        for (int i = 0; i < len; i++) {
            int ai = -1;
            for (int k = 0; k < A->nalpha; k++) if (A->alpha[k] == word[i]) ai = k;
            if (ai < 0) return 0;
            d = A->dnext[(size_t)d * A->nalpha + ai];
            if (d < 0) return 0;
        }
        return A->dfinal[d];
    }
    int cw = A->cw;
    uint64_t *cur = (uint64_t *)calloc(cw, 8), *nxt = (uint64_t *)calloc(cw, 8);
    memcpy(cur, A->closure + (size_t)A->tstart * cw, cw * 8);
    for (int i = 0; i < len; i++) {
        memset(nxt, 0, cw * 8);
        for (int q = 0; q < A->tn; q++) if (bs_test(cur, q))
            for (int k = A->tlab_off[q]; k < A->tlab_off[q + 1]; k++)
                if (A->tlab_label[k] == word[i]) {
                    const uint64_t *c = A->closure + (size_t)A->tlab_to[k] * cw;
                    for (int w = 0; w < cw; w++) nxt[w] |= c[w];
                }
        uint64_t *x = cur; cur = nxt; nxt = x;
    }
    int r = bs_test(cur, A->taccept);
    free(cur); free(nxt);
    return r;
}

/* ======================================================================
 * Per-source product-graph BFS, parallel over sources.
 * ====================================================================== */
typedef struct {
    const og_graph *g; const og_automaton *A; int use_dfa;
    const uint32_t *sources; uint64_t nsrc;
    int want_pairs;
    int64_t max_hops;           /* length bound: expand only nodes at depth < max_hops; -1 = none */
    uint64_t *counts, *pe;
    uint32_t **tlist;           /* per source sorted targets (want_pairs) */
    volatile uint64_t next;     /* dynamic chunking counter */
    int failed;
} job;

typedef struct { uint32_t v; int q; int64_t d; } pv;   /* product vertex (vertex, state), BFS depth */

static void *worker(void *arg) {
    job *J = (job *)arg;
    const og_graph *g = J->g; const og_automaton *A = J->A;
    int nq = J->use_dfa ? A->dn : A->tn;
    uint64_t nbits = (uint64_t)g->nv * (uint64_t)(nq ? nq : 1);
    uint64_t *vis = (uint64_t *)calloc((nbits + 63) / 64, 8);         /* visited set */
    uint64_t *tgt = (uint64_t *)calloc(((uint64_t)g->nv + 63) / 64, 8);  /* distinct targets */
    uint64_t qcap = 1024, tcap = 1024;
    pv *queue = (pv *)malloc(qcap * sizeof(pv));
    uint32_t *targets = (uint32_t *)malloc(tcap * sizeof(uint32_t));
    if (!vis || !tgt || !queue || !targets) { J->failed = 1; goto out; }
    for (;;) {
        uint64_t base = __atomic_fetch_add(&J->next, 16, __ATOMIC_RELAXED);
        if (base >= J->nsrc) break;
        uint64_t end = base + 16 < J->nsrc ? base + 16 : J->nsrc;
        for (uint64_t si = base; si < end; si++) {
            uint32_t x = J->sources[si];
            uint64_t qh = 0, qt = 0, nt = 0, pe = 0;
#define VISIT(V, Q, D) do {                                                     \
        uint64_t _b = (uint64_t)(V) * nq + (uint64_t)(Q);                        \
        if (!((vis[_b >> 6] >> (_b & 63)) & 1)) {                                \
            vis[_b >> 6] |= 1ull << (_b & 63);                                  \
            if (qt == qcap) { qcap *= 2; queue = (pv *)realloc(queue, qcap * sizeof(pv)); } \
            queue[qt].v = (V); queue[qt].q = (Q); queue[qt].d = (D); qt++;       \
        } } while (0)
            if (nq > 0) {
                if (J->use_dfa) {
                    VISIT(x, 0, 0);
                } else {
                    const uint64_t *c = A->closure + (size_t)A->tstart * A->cw;
                    for (int q = 0; q < A->tn; q++) if (bs_test(c, q)) VISIT(x, q, 0);
                }
            }
            while (qh < qt) {
                pv cur = queue[qh++];
                /* FIFO order = nondecreasing depth, so cur.d is the length of
                 * a shortest path to (cur.v, cur.q); with a bound, nodes at
                 * depth max_hops are reached (and may be final) but their
                 * out-edges are not traversed */
                const int expand = J->max_hops < 0 || cur.d < J->max_hops;
                int final_ = J->use_dfa ? A->dfinal[cur.q] : (cur.q == A->taccept);
                if (final_ && !((tgt[cur.v >> 6] >> (cur.v & 63)) & 1)) {
                    tgt[cur.v >> 6] |= 1ull << (cur.v & 63);
                    if (nt == tcap) { tcap *= 2; targets = (uint32_t *)realloc(targets, tcap * 4); }
                    targets[nt++] = cur.v;
                }
                if (!expand) continue;
                if (J->use_dfa) {
                    for (int ai = 0; ai < A->nalpha; ai++) {
                        int d2 = A->dnext[(size_t)cur.q * A->nalpha + ai];
                        if (d2 < 0) continue;
                        uint32_t l = (uint32_t)A->alpha[ai];
                        uint64_t s = (uint64_t)l * g->nv + cur.v;
                        pe += g->off[s + 1] - g->off[s];          /* product edges traversed */
                        for (uint64_t k = g->off[s]; k < g->off[s + 1]; k++) VISIT(g->adj[k], d2, cur.d + 1);
                    }
                } else {
                    for (int k = A->tlab_off[cur.q]; k < A->tlab_off[cur.q + 1]; k++) {
                        uint32_t l = (uint32_t)A->tlab_label[k];
                        const uint64_t *c = A->closure + (size_t)A->tlab_to[k] * A->cw;
                        uint64_t s = (uint64_t)l * g->nv + cur.v;
                        pe += g->off[s + 1] - g->off[s];
                        for (uint64_t e = g->off[s]; e < g->off[s + 1]; e++)
                            for (int q2 = 0; q2 < A->tn; q2++) if (bs_test(c, q2)) VISIT(g->adj[e], q2, cur.d + 1);
                    }
                }
            }
#undef VISIT
            /* reset the visited set through the queue (= touched list) */
            for (uint64_t i = 0; i < qt; i++) {
                uint64_t b = (uint64_t)queue[i].v * nq + (uint64_t)queue[i].q;
                vis[b >> 6] &= ~(1ull << (b & 63));
            }
            for (uint64_t i = 0; i < nt; i++) tgt[targets[i] >> 6] &= ~(1ull << (targets[i] & 63));
            J->counts[si] = nt;
            if (J->pe) J->pe[si] = pe;
            if (J->want_pairs) {
                uint32_t *lst = (uint32_t *)malloc((nt ? nt : 1) * 4);
                if (!lst) { J->failed = 1; continue; }
                memcpy(lst, targets, nt * 4);
                qsort(lst, nt, 4, cmp_u32);
                J->tlist[si] = lst;
            }
        }
    }
out:
    free(vis); free(tgt); free(queue); free(targets);
    return NULL;
}

/*
 * og_eval: evaluate for each sources[i] the single-source RPQ {(x, y)}.
 *   counts[i] = number of distinct y; pe[i] (optional) = product edges
 *   traversed (sum over reached (v,q) of out-degree in the product).
 *   want_pairs: *psrc and *pdst receive malloc'ed arrays of all pairs, sorted by
 *   (source order as given, y ascending); free with og_free.
 */
int og_eval_bounded(const og_graph *g, const og_automaton *A, int use_dfa,
                    const uint32_t *sources, uint64_t nsrc, int nthreads, int want_pairs, int64_t max_hops,
                    uint64_t *counts, uint64_t *pe, uint32_t **psrc, uint32_t **pdst, uint64_t *npairs) {
    for (uint64_t i = 0; i < nsrc; i++) if (sources[i] >= g->nv) return OG_EINVAL;
    job J; memset(&J, 0, sizeof(J));
    J.max_hops = max_hops;
    J.g = g; J.A = A; J.use_dfa = use_dfa; J.sources = sources; J.nsrc = nsrc;
    J.want_pairs = want_pairs; J.counts = counts; J.pe = pe;
    if (want_pairs) J.tlist = (uint32_t **)calloc(nsrc ? nsrc : 1, sizeof(uint32_t *));
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    for (int i = 0; i < nthreads; i++) pthread_create(&th[i], NULL, worker, &J);
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
    free(th);
    if (J.failed) return OG_ENOMEM;
    if (want_pairs) {
        uint64_t tot = 0;
        for (uint64_t i = 0; i < nsrc; i++) tot += counts[i];
        uint32_t *S = (uint32_t *)malloc((tot ? tot : 1) * 4), *D = (uint32_t *)malloc((tot ? tot : 1) * 4);
        uint64_t k = 0;
        for (uint64_t i = 0; i < nsrc; i++) {
            for (uint64_t j = 0; j < counts[i]; j++) { S[k] = sources[i]; D[k] = J.tlist[i][j]; k++; }
            free(J.tlist[i]);
        }
        free(J.tlist);
        *psrc = S; *pdst = D; *npairs = tot;
    }
    return OG_OK;
}

/* og_eval_bounded with max_hops = -1: no length bound (Definition 1) */
int og_eval(const og_graph *g, const og_automaton *A, int use_dfa,
            const uint32_t *sources, uint64_t nsrc, int nthreads, int want_pairs,
            uint64_t *counts, uint64_t *pe, uint32_t **psrc, uint32_t **pdst, uint64_t *npairs) {
    return og_eval_bounded(g, A, use_dfa, sources, nsrc, nthreads, want_pairs, -1, counts, pe, psrc, pdst, npairs);
}

void og_free(void *p) { free(p); }
