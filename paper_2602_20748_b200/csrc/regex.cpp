// rpq_compile: regular expression over edge labels -> automaton (host side).
//
// PAPER.md: the automata-based approach "exploits the automaton corresponding
// to the regular expression of the given RPQ"; Fig. 2(a) shows abc*
// as q0 -a-> q1 -b-> q2 with a c-loop on q2; Q4 abcd
// has |Q| = 5.  The route here is
//   tokenise (longest match, reading R3) -> parse (reading R2) ->
//   Glushkov position automaton (epsilon-free by construction) ->
//   subset construction -> Hopcroft minimisation -> trim -> canonical
//   BFS numbering,
// so the device traversal runs on the minimal trim DFA (the automaton the PE
// metric is defined on, reading R12).  If that DFA has more than
// RPQ_MAX_STATES states the trimmed Glushkov NFA is kept instead; the
// traversal kernels accept any epsilon-free automaton.
#include <algorithm>
#include <cstring>
#include <deque>
#include <map>
#include <set>

#include "internal.h"

namespace {

enum Kind { K_LABEL, K_CAT, K_ALT, K_STAR, K_PLUS, K_OPT };
struct Node {
    Kind k;
    int label;   // K_LABEL
    int a, b;    // children (-1 none)
};

struct Tok {
    int type;    // 0 = label, 1 = operator, 2 = end
    int label;
    char op;
    size_t off;
};

struct Parser {
    std::vector<Tok> toks;
    size_t i = 0;
    bool paper = false;
    std::vector<Node> nodes;
    rpq_status st = RPQ_OK;
    size_t err_off = 0;

    const Tok &peek() const { return toks[i]; }
    bool is_op(char c) const { return peek().type == 1 && peek().op == c; }
    int add(Node n) { nodes.push_back(n); return (int)nodes.size() - 1; }
    void fail(rpq_status s) { if (st == RPQ_OK) { st = s; err_off = peek().off; } }

    int alt() {
        int r = cat();
        while (st == RPQ_OK && (is_op('|') || (paper && is_op('+')))) {
            ++i;
            int q = cat();
            r = add({K_ALT, -1, r, q});
        }
        return r;
    }
    bool starts_atom() const { return peek().type == 0 || (peek().type == 1 && peek().op == '('); }
    int cat() {
        int r = post();
        while (st == RPQ_OK && starts_atom()) {
            int q = post();
            r = add({K_CAT, -1, r, q});
        }
        return r;
    }
    int post() {
        int r = atom();
        while (st == RPQ_OK) {
            if (is_op('*')) r = add({K_STAR, -1, r, -1});
            else if (is_op('?')) r = add({K_OPT, -1, r, -1});
            else if (!paper && is_op('+')) r = add({K_PLUS, -1, r, -1});
            else break;
            ++i;
        }
        return r;
    }
    int atom() {
        if (st != RPQ_OK) return -1;
        if (peek().type == 0) return add({K_LABEL, toks[i++].label, -1, -1});
        if (is_op('(')) {
            ++i;
            int r = alt();
            if (st != RPQ_OK) return -1;
            if (!is_op(')')) { fail(RPQ_ESYNTAX); return -1; }
            ++i;
            return r;
        }
        fail(RPQ_ESYNTAX);
        return -1;
    }
};

rpq_status tokenize(const std::vector<std::string> &vocab, const char *s, std::vector<Tok> &out,
                    size_t *err_off) {
    size_t n = std::strlen(s), p = 0;
    while (p < n) {
        char c = s[p];
        if (c == ' ' || c == '\t' || c == '\n' || c == '.' || c == '/') { ++p; continue; }
        if (std::strchr("()|*+?", c)) { out.push_back({1, -1, c, p}); ++p; continue; }
        int best = -1;
        size_t bl = 0;
        for (size_t k = 0; k < vocab.size(); ++k) {
            const std::string &nm = vocab[k];
            if (!nm.empty() && nm.size() > bl && nm.size() <= n - p && !nm.compare(0, nm.size(), s + p, nm.size())) {
                best = (int)k;
                bl = nm.size();
            }
        }
        if (best < 0) { *err_off = p; return RPQ_ELABEL; }
        out.push_back({0, best, 0, p});
        p += bl;
    }
    out.push_back({2, -1, 0, n});
    return RPQ_OK;
}

// ---- Glushkov position automaton ----------------------------------------
using Bits = std::vector<uint64_t>;
struct Glushkov {
    int npos = 0;                          // positions 1..npos; state 0 initial
    std::vector<int> pos_label;            // [npos+1]
    std::vector<Bits> follow;              // [npos+1]
    Bits first, last;
    bool nullable = false;
};

static void bset(Bits &b, int i) { b[i >> 6] |= 1ull << (i & 63); }
static bool btest(const Bits &b, int i) { return (b[i >> 6] >> (i & 63)) & 1; }
static void bor(Bits &a, const Bits &b) { for (size_t k = 0; k < a.size(); ++k) a[k] |= b[k]; }

struct GInfo { bool nullable; Bits first, last; };

GInfo glushkov_rec(const std::vector<Node> &nodes, int idx, Glushkov &G, int W) {
    const Node &n = nodes[idx];
    GInfo r{false, Bits(W, 0), Bits(W, 0)};
    switch (n.k) {
    case K_LABEL: {
        int p = ++G.npos;
        G.pos_label[p] = n.label;
        bset(r.first, p); bset(r.last, p);
        break;
    }
    case K_ALT: {
        GInfo a = glushkov_rec(nodes, n.a, G, W), b = glushkov_rec(nodes, n.b, G, W);
        r.nullable = a.nullable || b.nullable;
        r.first = a.first; bor(r.first, b.first);
        r.last = a.last; bor(r.last, b.last);
        break;
    }
    case K_CAT: {
        GInfo a = glushkov_rec(nodes, n.a, G, W), b = glushkov_rec(nodes, n.b, G, W);
        r.nullable = a.nullable && b.nullable;
        r.first = a.first; if (a.nullable) bor(r.first, b.first);
        r.last = b.last; if (b.nullable) bor(r.last, a.last);
        for (int p = 1; p <= G.npos; ++p) if (btest(a.last, p)) bor(G.follow[p], b.first);
        break;
    }
    case K_STAR: case K_PLUS: case K_OPT: {
        GInfo a = glushkov_rec(nodes, n.a, G, W);
        r.nullable = (n.k == K_PLUS) ? a.nullable : true;
        r.first = a.first; r.last = a.last;
        if (n.k != K_OPT)
            for (int p = 1; p <= G.npos; ++p) if (btest(a.last, p)) bor(G.follow[p], a.first);
        break;
    }
    }
    return r;
}

// An explicit automaton used between stages: states 0..n-1, initial 0.
struct Auto {
    int n = 0;
    std::vector<std::vector<std::pair<int, int>>> out;   // (label, to)
    std::vector<char> fin;
};

// Trim (reachable from 0 AND co-reachable to a final) + canonical BFS
// numbering (successors visited in (label, to) order).
Auto trim_canon(const Auto &A) {
    std::vector<char> reach(A.n, 0), co(A.n, 0);
    std::deque<int> dq;
    if (A.n) { reach[0] = 1; dq.push_back(0); }
    while (!dq.empty()) {
        int x = dq.front(); dq.pop_front();
        for (auto &e : A.out[x]) if (!reach[e.second]) { reach[e.second] = 1; dq.push_back(e.second); }
    }
    std::vector<std::vector<int>> in(A.n);
    for (int x = 0; x < A.n; ++x) for (auto &e : A.out[x]) in[e.second].push_back(x);
    for (int x = 0; x < A.n; ++x) if (A.fin[x]) { co[x] = 1; dq.push_back(x); }
    while (!dq.empty()) {
        int x = dq.front(); dq.pop_front();
        for (int y : in[x]) if (!co[y]) { co[y] = 1; dq.push_back(y); }
    }
    std::vector<int> id(A.n, -1), order;
    if (A.n && reach[0] && co[0]) { id[0] = 0; order.push_back(0); }
    for (size_t h = 0; h < order.size(); ++h) {
        int x = order[h];
        auto es = A.out[x];
        std::sort(es.begin(), es.end());
        for (auto &e : es) {
            int y = e.second;
            if (reach[y] && co[y] && id[y] < 0) { id[y] = (int)order.size(); order.push_back(y); }
        }
    }
    Auto R;
    R.n = (int)order.size();
    R.out.resize(R.n);
    R.fin.assign(R.n, 0);
    for (int i = 0; i < R.n; ++i) {
        int x = order[i];
        R.fin[i] = A.fin[x];
        for (auto &e : A.out[x]) if (id[e.second] >= 0) R.out[i].push_back({e.first, id[e.second]});
        std::sort(R.out[i].begin(), R.out[i].end());
        R.out[i].erase(std::unique(R.out[i].begin(), R.out[i].end()), R.out[i].end());
    }
    return R;
}

// Subset construction over the Glushkov automaton; returns false if more
// than `cap` DFA states would be needed.
bool subset(const Auto &N, const std::vector<int> &alpha, int cap, Auto &D) {
    int W = (N.n + 63) / 64;
    std::map<Bits, int> idx;
    std::vector<Bits> sets;
    Bits s0(W, 0); bset(s0, 0);
    idx[s0] = 0; sets.push_back(s0);
    D = Auto();
    D.out.emplace_back();
    for (size_t d = 0; d < sets.size(); ++d) {
        for (int l : alpha) {
            Bits t(W, 0);
            bool any = false;
            for (int q = 0; q < N.n; ++q) if (btest(sets[d], q))
                for (auto &e : N.out[q]) if (e.first == l) { bset(t, e.second); any = true; }
            if (!any) continue;
            auto it = idx.find(t);
            int tid;
            if (it == idx.end()) {
                if ((int)sets.size() >= cap) return false;
                tid = (int)sets.size();
                idx[t] = tid; sets.push_back(t); D.out.emplace_back();
            } else tid = it->second;
            D.out[d].push_back({l, tid});
        }
    }
    D.n = (int)sets.size();
    D.fin.assign(D.n, 0);
    for (int d = 0; d < D.n; ++d)
        for (int q = 0; q < N.n; ++q) if (btest(sets[d], q) && N.fin[q]) { D.fin[d] = 1; break; }
    return true;
}

// Hopcroft partition refinement on the DFA completed with a dead state.
Auto hopcroft(const Auto &D, const std::vector<int> &alpha) {
    int n = D.n + 1, dead = D.n, k = (int)alpha.size();
    std::vector<int> delta((size_t)n * k, dead);
    for (int d = 0; d < D.n; ++d)
        for (auto &e : D.out[d]) {
            int a = (int)(std::find(alpha.begin(), alpha.end(), e.first) - alpha.begin());
            delta[(size_t)d * k + a] = e.second;
        }
    std::vector<std::vector<int>> inv((size_t)n * k);
    for (int d = 0; d < n; ++d) for (int a = 0; a < k; ++a) inv[(size_t)delta[(size_t)d * k + a] * k + a].push_back(d);
    std::vector<int> block(n);
    std::vector<std::vector<int>> blocks;
    std::vector<int> F, NF;
    for (int d = 0; d < n; ++d) ((d < D.n && D.fin[d]) ? F : NF).push_back(d);
    std::set<std::pair<int, int>> work;   // (block, symbol)
    for (auto *B : {&F, &NF}) if (!B->empty()) {
        for (int d : *B) block[d] = (int)blocks.size();
        blocks.push_back(*B);
    }
    if (blocks.size() == 2) {
        int small = blocks[0].size() <= blocks[1].size() ? 0 : 1;
        for (int a = 0; a < k; ++a) work.insert({small, a});
    }
    while (!work.empty()) {
        auto [A, c] = *work.begin();
        work.erase(work.begin());
        std::vector<char> inX(n, 0);
        for (int t : blocks[A]) for (int s : inv[(size_t)t * k + c]) inX[s] = 1;
        std::set<int> touched;
        for (int s = 0; s < n; ++s) if (inX[s]) touched.insert(block[s]);
        for (int Y : touched) {
            std::vector<int> y1, y2;
            for (int s : blocks[Y]) (inX[s] ? y1 : y2).push_back(s);
            if (y1.empty() || y2.empty()) continue;
            int Ynew = (int)blocks.size();
            blocks[Y] = y1;
            blocks.push_back(y2);
            for (int s : y2) block[s] = Ynew;
            for (int a = 0; a < k; ++a) {
                if (work.count({Y, a})) work.insert({Ynew, a});
                else work.insert({blocks[Y].size() <= blocks[Ynew].size() ? Y : Ynew, a});
            }
        }
    }
    // quotient, with the initial state's block first
    Auto Q;
    Q.n = (int)blocks.size();
    Q.out.resize(Q.n);
    Q.fin.assign(Q.n, 0);
    std::vector<int> remap(Q.n, -1);
    remap[block[0]] = 0;
    int nid = 1;
    for (int b = 0; b < Q.n; ++b) if (remap[b] < 0) remap[b] = nid++;
    for (int b = 0; b < Q.n; ++b) {
        int rep = blocks[b][0];
        int qb = remap[b];
        Q.fin[qb] = rep < D.n && D.fin[rep];
        for (int a = 0; a < k; ++a) Q.out[qb].push_back({alpha[a], remap[block[delta[(size_t)rep * k + a]]]});
    }
    return Q;   // the dead block is removed by trim_canon (not co-reachable)
}

// Final stage shared by rpq_compile and rpq_nfa_reverse: the trimmed,
// canonically numbered automaton -> rpq_nfa (limits of the kernels checked).
rpq_status make_nfa(const Auto &R, bool is_dfa, const std::vector<std::string> &vocab, rpq_nfa **out) {
    if (R.n > RPQ_MAX_STATES)
        return rpq_fail(RPQ_EUNSUPPORTED, "rpq_compile: %d automaton states > %d", R.n, RPQ_MAX_STATES);
    rpq_nfa *a = new rpq_nfa();
    a->nq = (uint32_t)R.n;
    a->is_dfa = is_dfa;
    a->vocab = vocab;
    a->vocab_size = (uint32_t)vocab.size();
    a->off.assign(a->nq + 1, 0);
    std::set<uint32_t> labs;
    for (int q = 0; q < R.n; ++q) {
        if (R.fin[q]) a->final_mask |= 1ull << q;
        for (auto &e : R.out[q]) {
            a->from.push_back((uint32_t)q);
            a->label.push_back((uint32_t)e.first);
            a->to.push_back((uint32_t)e.second);
            labs.insert((uint32_t)e.first);
        }
        a->off[q + 1] = (uint32_t)a->from.size();
    }
    a->accepts_empty = R.n > 0 && R.fin[0];
    if (a->from.size() > RPQ_MAX_TRANSITIONS || labs.size() > RPQ_MAX_QUERY_LABELS) {
        delete a;
        return rpq_fail(RPQ_EUNSUPPORTED, "rpq_compile: automaton too large for the kernels");
    }
    *out = a;
    return RPQ_OK;
}

}  // namespace

rpq_status compile_regex(const std::vector<std::string> &vocab, const char *regex, uint32_t flags,
                         rpq_nfa **out, size_t *err_offset) {
    if (out) *out = nullptr;
    if (err_offset) *err_offset = 0;
    if (!regex || !out) return rpq_fail(RPQ_EINVAL, "rpq_compile: NULL argument");
    Parser P;
    P.paper = (flags & RPQ_SYNTAX_PAPER) != 0;
    size_t eo = 0;
    rpq_status st = tokenize(vocab, regex, P.toks, &eo);
    if (st != RPQ_OK) {
        if (err_offset) *err_offset = eo;
        return rpq_fail(st, "rpq_compile: unknown label at offset %zu in '%s'", eo, regex);
    }
    int root = P.alt();
    if (P.st == RPQ_OK && P.peek().type != 2) P.fail(RPQ_ESYNTAX);
    if (P.st != RPQ_OK) {
        if (err_offset) *err_offset = P.err_off;
        return rpq_fail(P.st, "rpq_compile: syntax error at offset %zu in '%s'", P.err_off, regex);
    }
    // Glushkov
    int nlab = 0;
    for (auto &n : P.nodes) nlab += n.k == K_LABEL;
    int W = (nlab + 1 + 63) / 64;
    Glushkov G;
    G.pos_label.assign(nlab + 1, -1);
    G.follow.assign(nlab + 1, Bits(W, 0));
    GInfo gi = glushkov_rec(P.nodes, root, G, W);
    Auto N;
    N.n = nlab + 1;
    N.out.resize(N.n);
    N.fin.assign(N.n, 0);
    N.fin[0] = gi.nullable;
    for (int p = 1; p <= nlab; ++p) {
        if (btest(gi.first, p)) N.out[0].push_back({G.pos_label[p], p});
        if (btest(gi.last, p)) N.fin[p] = 1;
        for (int p2 = 1; p2 <= nlab; ++p2) if (btest(G.follow[p], p2)) N.out[p].push_back({G.pos_label[p2], p2});
    }
    std::vector<int> alpha;
    for (int p = 1; p <= nlab; ++p) alpha.push_back(G.pos_label[p]);
    std::sort(alpha.begin(), alpha.end());
    alpha.erase(std::unique(alpha.begin(), alpha.end()), alpha.end());

    Auto R;
    bool is_dfa = false;
    Auto D;
    if (!(flags & RPQ_NO_MINIMIZE) && subset(N, alpha, 4096, D)) {
        Auto M = trim_canon(hopcroft(D, alpha));
        if (M.n <= RPQ_MAX_STATES) { R = M; is_dfa = true; }
    }
    if (!is_dfa) R = trim_canon(N);
    return make_nfa(R, is_dfa, vocab, out);
}

// Reversed language (rpq_nfa_reverse): reverse every transition of the
// epsilon-free automaton, a new initial state 0 takes the reversed
// transitions into the old final states (so no epsilon moves are needed), the
// old initial state becomes final (and 0 too when epsilon is accepted); then
// the same determinise / minimise / trim / number pipeline as rpq_compile.
rpq_status reverse_automaton(const rpq_nfa *a, rpq_nfa **out) {
    if (out) *out = nullptr;
    if (!a || !out) return rpq_fail(RPQ_EINVAL, "rpq_nfa_reverse: NULL argument");
    Auto N;
    N.n = (int)a->nq + 1;
    N.out.resize(N.n);
    N.fin.assign(N.n, 0);
    std::vector<int> alpha;
    for (size_t t = 0; t < a->from.size(); ++t) {
        const int q = (int)a->from[t], l = (int)a->label[t], q2 = (int)a->to[t];
        N.out[q2 + 1].push_back({l, q + 1});
        if ((a->final_mask >> q2) & 1ull) N.out[0].push_back({l, q + 1});
        alpha.push_back(l);
    }
    if (a->nq) N.fin[1] = 1;               // the old initial state
    N.fin[0] = a->accepts_empty;
    std::sort(alpha.begin(), alpha.end());
    alpha.erase(std::unique(alpha.begin(), alpha.end()), alpha.end());
    Auto R, D;
    bool is_dfa = false;
    if (subset(N, alpha, 4096, D)) {
        Auto M = trim_canon(hopcroft(D, alpha));
        if (M.n <= RPQ_MAX_STATES) { R = M; is_dfa = true; }
    }
    if (!is_dfa) R = trim_canon(N);
    return make_nfa(R, is_dfa, a->vocab, out);
}
