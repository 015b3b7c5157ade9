// Data-affinity-based reordering, Algorithm 1 (§3.2).
//
// Step I (Alg. 1 l.1-8): vertices of the affinity graph G = pattern(A or A^T)
// minus the diagonal are visited once in ascending degree (ties by
// id); each is merged into the neighbouring community u maximising the merge
// gain dQ(u,v) = 2*(w_uv/2m - a_u*a_v/(2m)^2) (Eq. 1 read as a merge
// differential) if dQ > 0 (ties: smallest community id).  Community
// edge lists are aggregated lazily (coarsening) and compacted when a community
// is visited.  Step II (l.9-27): DFS over the merge forest (roots ascending,
// node before children, children in merge order) gives the leaf sequence; each
// unvisited vertex v gets the next id, then the walk repeatedly jumps to the
// vertex with the most common neighbours among the next L = 64 unvisited
// vertices in DFS order (neighbour lists capped at H = 128 entries), ties by DFS
// order; with no common neighbour it resumes the DFS sequence (Q13).
// Reading R6b: after a visit, a community passes on at most its 256
// heaviest neighbour-community edges, so chains of merges on meshes stay O(m).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "../internal.hpp"

namespace accspmm {

namespace {

int env_or(const char *name, int dflt)
{
    const char *s = std::getenv(name);
    return s ? std::atoi(s) : dflt;
}

// ACCSPMM_TRACE=1: phase times of the reordering on stderr
struct Trace {
    bool on = env_or("ACCSPMM_TRACE", 0) != 0;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char *what)
    {
        if (!on) return;
        auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[accspmm reorder] %-28s %9.1f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};
constexpr size_t kEdgeCap = 256;  // community edges carried up a merge (reading R6b)

struct Graph {
    std::vector<int64_t> ptr;
    std::vector<uint32_t> adj;
};

// pattern(A or A^T) without the diagonal, as sorted unique adjacency lists.  A
// structurally symmetric A (the graph workloads) is its own affinity graph: checked in
// parallel by binary search, then copied without the diagonal.  Otherwise A and A^T are
// merged by a counting scatter and every list is sorted and deduplicated.
Graph affinity_graph(const Csr &a)
{
    const int64_t n = a.M;
    bool sym = true;
#pragma omp parallel for schedule(dynamic, 1024) reduction(&& : sym)
    for (int64_t i = 0; i < n; ++i) {
        if (!sym) continue;
        for (int64_t p = a.rowptr[i]; p < a.rowptr[i + 1] && sym; ++p) {
            const int64_t j = a.colidx[p];
            if (j == i) continue;
            const int32_t *b = a.colidx + a.rowptr[j], *e = a.colidx + a.rowptr[j + 1];
            sym = std::binary_search(b, e, (int32_t)i);
        }
    }
    Graph g;
    g.ptr.assign((size_t)n + 1, 0);
    if (sym) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            const int32_t *b = a.colidx + a.rowptr[i], *e = a.colidx + a.rowptr[i + 1];
            g.ptr[(size_t)i + 1] = (e - b) - (std::binary_search(b, e, (int32_t)i) ? 1 : 0);
        }
        for (int64_t i = 0; i < n; ++i) g.ptr[(size_t)i + 1] += g.ptr[(size_t)i];
        g.adj.resize((size_t)g.ptr[(size_t)n]);
#pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t i = 0; i < n; ++i) {
            size_t q = (size_t)g.ptr[(size_t)i];
            for (int64_t p = a.rowptr[i]; p < a.rowptr[i + 1]; ++p)
                if (a.colidx[p] != i) g.adj[q++] = (uint32_t)a.colidx[p];
        }
        return g;
    }
    std::vector<int64_t> cnt((size_t)n + 1, 0);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = a.rowptr[i]; p < a.rowptr[i + 1]; ++p) {
            int64_t j = a.colidx[p];
            if (j == i) continue;
            cnt[(size_t)i + 1]++;
            cnt[(size_t)j + 1]++;
        }
    for (int64_t i = 0; i < n; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i];
    std::vector<uint32_t> tmp((size_t)cnt[(size_t)n]);
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = a.rowptr[i]; p < a.rowptr[i + 1]; ++p) {
            int64_t j = a.colidx[p];
            if (j == i) continue;
            tmp[(size_t)fill[(size_t)i]++] = (uint32_t)j;
            tmp[(size_t)fill[(size_t)j]++] = (uint32_t)i;
        }
    std::vector<int64_t> uniq((size_t)n, 0);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        auto b = tmp.begin() + cnt[(size_t)i], e = tmp.begin() + cnt[(size_t)i + 1];
        std::sort(b, e);
        uniq[(size_t)i] = std::unique(b, e) - b;
    }
    for (int64_t i = 0; i < n; ++i) g.ptr[(size_t)i + 1] = g.ptr[(size_t)i] + uniq[(size_t)i];
    g.adj.resize((size_t)g.ptr[(size_t)n]);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i)
        std::copy(tmp.begin() + cnt[(size_t)i], tmp.begin() + cnt[(size_t)i] + uniq[(size_t)i],
                  g.adj.begin() + g.ptr[(size_t)i]);
    return g;
}

}  // namespace

std::vector<uint32_t> reorder_alg1(const Csr &a)
{
    const int64_t n = a.M;
    std::vector<uint32_t> perm((size_t)n);
    std::iota(perm.begin(), perm.end(), 0u);
    if (n == 0 || a.M != a.K) return perm;  // Q14: non-square -> identity
    Trace tr;
    Graph g = affinity_graph(a);
    tr.mark("affinity graph");
    const double m2 = (double)g.ptr[(size_t)n];

    // ---------------- Step I: dendrogram construction (one pass) ----------------
    std::vector<uint32_t> parent((size_t)n);
    std::iota(parent.begin(), parent.end(), 0u);
    // per community: its degree sum a_c (Eq. 1) and the edge weight accumulated towards the
    // vertex being visited, side by side so the merge-gain loop reads one cache line
    struct Comm {
        uint64_t w;
        double a;
    };
    std::vector<Comm> cm((size_t)n, Comm{0, 0.0});
    std::vector<uint32_t> first_child((size_t)n, UINT32_MAX), last_child((size_t)n, UINT32_MAX),
        next_sib((size_t)n, UINT32_MAX);
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> E((size_t)n);
    std::vector<uint32_t> order((size_t)n);
    std::iota(order.begin(), order.end(), 0u);
    for (int64_t v = 0; v < n; ++v) cm[(size_t)v].a = (double)(g.ptr[(size_t)v + 1] - g.ptr[(size_t)v]);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
        return g.ptr[x + 1] - g.ptr[x] < g.ptr[y + 1] - g.ptr[y];
    });
    auto find = [&](uint32_t x) {
        uint32_t r = x;
        while (parent[r] != r) r = parent[r];
        while (parent[x] != r) { uint32_t nx = parent[x]; parent[x] = r; x = nx; }
        return r;
    };
    std::vector<uint32_t> touched;
    for (uint32_t v : order) {
        const int64_t deg = g.ptr[v + 1] - g.ptr[v];
        if (deg == 0 || m2 == 0.0) continue;
        touched.clear();
        auto add = [&](uint32_t x, uint32_t w) {
            uint32_t r = find(x);
            if (r == v) return;
            if (cm[r].w == 0) touched.push_back(r);
            cm[r].w += w;
        };
        for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
            if (p + 16 < g.ptr[v + 1]) {  // the walk is bound by random accesses: prefetch ahead
                const uint32_t x = g.adj[(size_t)p + 16];
                __builtin_prefetch(&parent[x]);
                __builtin_prefetch(&cm[x], 1);
            }
            add(g.adj[(size_t)p], 1u);
        }
        for (size_t q = 0; q < E[v].size(); ++q) {
            if (q + 16 < E[v].size()) __builtin_prefetch(&parent[E[v][q + 16].first]);
            add(E[v][q].first, E[v][q].second);
        }
        // touched is in first-touch order: the argmax breaks ties by the smallest id explicitly,
        // and every later use of comp is order-independent (integer sums, a total-order cut)
        std::vector<std::pair<uint32_t, uint32_t>> comp;
        comp.reserve(touched.size());
        uint32_t best = UINT32_MAX;
        double best_dq = 0.0;
        for (uint32_t r : touched) {
            double dq = 2.0 * ((double)cm[r].w / m2 - cm[r].a * cm[v].a / (m2 * m2));
            if (best == UINT32_MAX || dq > best_dq || (dq == best_dq && r < best)) { best = r; best_dq = dq; }
            comp.emplace_back(r, (uint32_t)cm[r].w);
            cm[r].w = 0;
        }
        E[v].clear();
        E[v].shrink_to_fit();
        // R6b: only the kEdgeCap heaviest community edges (ties: smaller id) are carried on,
        // which bounds the coarsening work on meshes; the merge decision above is exact.
        if (comp.size() > kEdgeCap) {
            std::partial_sort(comp.begin(), comp.begin() + kEdgeCap, comp.end(),
                              [](const std::pair<uint32_t, uint32_t> &x, const std::pair<uint32_t, uint32_t> &y) {
                                  return x.second != y.second ? x.second > y.second : x.first < y.first;
                              });
            comp.resize(kEdgeCap);
        }
        if (best != UINT32_MAX && best_dq > 0.0) {
            const uint32_t u = best;
            parent[v] = u;
            cm[u].a += cm[v].a;
            // v's original edges were consumed into comp; u inherits the aggregated list
            E[u].insert(E[u].end(), comp.begin(), comp.end());
            if (first_child[u] == UINT32_MAX) first_child[u] = v; else next_sib[last_child[u]] = v;
            last_child[u] = v;
        } else {
            // v stays a root: keep its compacted list for communities merging into it later
            E[v] = std::move(comp);
        }
    }
    // A vertex is visited exactly once; its graph adjacency is read only on that
    // visit, and afterwards its aggregated edges live in E[] of itself or its parent.
    tr.mark("step I (dendrogram)");

    // ---------------- Step II: ordering generation ----------------
    std::vector<uint32_t> seq;
    seq.reserve((size_t)n);
    std::vector<uint32_t> stack;
    for (int64_t r = 0; r < n; ++r) {
        if (parent[(size_t)r] != (uint32_t)r) continue;
        stack.push_back((uint32_t)r);
        while (!stack.empty()) {
            uint32_t x = stack.back();
            stack.pop_back();
            seq.push_back(x);
            // push children in reverse merge order so they pop in merge order
            std::vector<uint32_t> ch;
            for (uint32_t c = first_child[x]; c != UINT32_MAX; c = next_sib[c]) ch.push_back(c);
            for (auto it = ch.rbegin(); it != ch.rend(); ++it) stack.push_back(*it);
        }
    }
    // doubly linked list of unvisited positions in seq
    std::vector<int64_t> nxt((size_t)n + 1), prv((size_t)n + 1);
    std::vector<int64_t> pos_of((size_t)n);
    for (int64_t i = 0; i < n; ++i) pos_of[seq[(size_t)i]] = i;
    // sentinel at index n
    for (int64_t i = 0; i <= n; ++i) { nxt[(size_t)i] = i + 1; prv[(size_t)i] = i - 1; }
    nxt[(size_t)n] = 0;
    prv[0] = n;
    prv[(size_t)n] = n - 1;
    if (n > 0) nxt[(size_t)n - 1] = n;
    const int L = knobs().reorder_L, H = knobs().reorder_H;  // reading R6 (variants build: sweepable)
    std::vector<char> visited((size_t)n, 0);
    std::vector<uint32_t> mark((size_t)n, 0);
    uint32_t stamp = 0;
    int64_t next_id = 0;
    auto assign = [&](uint32_t x) {
        visited[x] = 1;
        perm[(size_t)next_id++] = x;
        int64_t p = pos_of[x];
        nxt[(size_t)prv[(size_t)p]] = nxt[(size_t)p];
        prv[(size_t)nxt[(size_t)p]] = prv[(size_t)p];
    };
    for (int64_t i = 0; i < n; ++i) {
        uint32_t v = seq[(size_t)i];
        if (visited[v]) continue;
        assign(v);
        while (nxt[(size_t)n] != n) {
            ++stamp;
            if (stamp == 0) { std::fill(mark.begin(), mark.end(), 0u); stamp = 1; }
            const int64_t dv = std::min<int64_t>(H, g.ptr[v + 1] - g.ptr[v]);
            for (int64_t q = 0; q < dv; ++q) mark[g.adj[(size_t)(g.ptr[v] + q)]] = stamp;
            uint32_t best = UINT32_MAX;
            int64_t best_c = 0;
            int cand = 0;
            for (int64_t p = nxt[(size_t)n]; p != n && cand < L; p = nxt[(size_t)p], ++cand) {
                uint32_t u = seq[(size_t)p];
                const int64_t du = std::min<int64_t>(H, g.ptr[u + 1] - g.ptr[u]);
                int64_t c = 0;
                for (int64_t q = 0; q < du; ++q) c += mark[g.adj[(size_t)(g.ptr[u] + q)]] == stamp;
                if (c > best_c) { best_c = c; best = u; }
            }
            if (best == UINT32_MAX) break;
            assign(best);
            v = best;
        }
    }
    tr.mark("step II (ordering)");
    return perm;
}

}  // namespace accspmm
