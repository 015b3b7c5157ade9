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
#include <memory>
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

// adjacency storage without std::vector's serial zero fill (3.2B entries on papers100M)
struct U32Buf {
    std::unique_ptr<uint32_t[]> p;
    size_t n = 0;
    void resize(size_t m)
    {
        p.reset(new uint32_t[m ? m : 1]);
        n = m;
    }
    uint32_t &operator[](size_t i) { return p[i]; }
    const uint32_t &operator[](size_t i) const { return p[i]; }
    uint32_t *begin() { return p.get(); }
};

struct Graph {
    std::vector<int64_t> ptr;
    U32Buf adj;
};

// pattern(A or A^T) without the diagonal, as sorted unique adjacency lists.  A
// structurally symmetric A (the graph workloads) is its own affinity graph: checked in
// parallel by binary search, then copied without the diagonal.  Otherwise A and A^T are
// merged by a counting scatter and every list is sorted and deduplicated.
Graph affinity_graph(const Csr &a)
{
    const int64_t n = a.M;
    Trace tr;
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
    tr.mark("  symmetry check");
    // A or A^T: per row its own columns, then the rows that point at it.  The reverse entries
    // go through a bucketed transpose (destination buckets of 2^14 rows): each row chunk writes
    // its (destination, source) pairs into its slice of every bucket, then every bucket is
    // placed with cache-resident cursors -- no atomics and no random writes over the whole
    // array; each list is then sorted and deduplicated (so the entry order is immaterial).
    constexpr int kBucketShift = 14;
    const int64_t nbuck = (n >> kBucketShift) + 1;
    const int64_t nchunk = 256, chunk = (n + nchunk - 1) / nchunk;
    std::vector<int64_t> cnt((size_t)n + 1, 0), indeg((size_t)n, 0);
    std::vector<int64_t> bc((size_t)(nchunk * nbuck), 0);  // [chunk][bucket] pair counts
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nchunk; ++c) {
        int64_t *row = bc.data() + c * nbuck;
        for (int64_t i = c * chunk; i < std::min<int64_t>(n, (c + 1) * chunk); ++i) {
            int64_t own = 0;
            for (int64_t p = a.rowptr[i]; p < a.rowptr[i + 1]; ++p) {
                const int64_t j = a.colidx[p];
                if (j == i) continue;
                ++own;
                ++row[j >> kBucketShift];
            }
            cnt[(size_t)i + 1] = own;
        }
    }
    // bucket-major offsets of the pair array
    std::vector<int64_t> boff((size_t)(nchunk * nbuck) + 1, 0);
    {
        int64_t o = 0;
        for (int64_t bk = 0; bk < nbuck; ++bk)
            for (int64_t c = 0; c < nchunk; ++c) {
                boff[(size_t)(c * nbuck + bk)] = o;
                o += bc[(size_t)(c * nbuck + bk)];
            }
        boff[(size_t)(nchunk * nbuck)] = o;
    }
    const int64_t npairs = boff[(size_t)(nchunk * nbuck)];
    std::unique_ptr<uint64_t[]> pairs(new uint64_t[(size_t)std::max<int64_t>(npairs, 1)]);  // dst << 32 | src
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nchunk; ++c) {
        std::vector<int64_t> cur(boff.begin() + c * nbuck, boff.begin() + (c + 1) * nbuck);
        for (int64_t i = c * chunk; i < std::min<int64_t>(n, (c + 1) * chunk); ++i)
            for (int64_t p = a.rowptr[i]; p < a.rowptr[i + 1]; ++p) {
                const int64_t j = a.colidx[p];
                if (j == i) continue;
                pairs[(size_t)cur[(size_t)(j >> kBucketShift)]++] = ((uint64_t)j << 32) | (uint64_t)i;
            }
    }
    // in-degrees per bucket (cache resident), then row offsets
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t bk = 0; bk < nbuck; ++bk) {
        const int64_t p0 = boff[(size_t)bk], p1 = bk + 1 < nbuck ? boff[(size_t)(bk + 1)] : npairs;
        for (int64_t q = p0; q < p1; ++q) ++indeg[(size_t)(pairs[(size_t)q] >> 32)];
    }
    for (int64_t i = 0; i < n; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i] + indeg[(size_t)i];
    tr.mark("  counts");
    std::unique_ptr<uint32_t[]> tmp(new uint32_t[(size_t)std::max<int64_t>(cnt[(size_t)n], 1)]);  // no zero fill
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
        int64_t q = cnt[(size_t)i];
        for (int64_t p = a.rowptr[i]; p < a.rowptr[i + 1]; ++p)
            if (a.colidx[p] != i) tmp[(size_t)q++] = (uint32_t)a.colidx[p];
        indeg[(size_t)i] = q;  // reverse-entry cursor of row i
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t bk = 0; bk < nbuck; ++bk) {
        const int64_t p0 = boff[(size_t)bk], p1 = bk + 1 < nbuck ? boff[(size_t)(bk + 1)] : npairs;
        for (int64_t q = p0; q < p1; ++q) {
            const uint64_t e = pairs[(size_t)q];
            tmp[(size_t)indeg[(size_t)(e >> 32)]++] = (uint32_t)(e & 0xFFFFFFFFu);
        }
    }
    pairs.reset();
    std::vector<int64_t> fill;
    tr.mark("  scatter");
    // row i = its own columns (ascending: canonical CSR) followed by the rows pointing at it,
    // which arrive in ascending source order (buckets keep the chunk-major row order): one
    // merge of two sorted runs with deduplication instead of a sort
    std::vector<int64_t> uniq((size_t)n, 0);
#pragma omp parallel
    {
        std::vector<uint32_t> buf;
#pragma omp for schedule(dynamic, 1024)
        for (int64_t i = 0; i < n; ++i) {
            uint32_t *b = tmp.get() + cnt[(size_t)i], *e = tmp.get() + cnt[(size_t)i + 1];
            const int32_t *rb = a.colidx + a.rowptr[i], *re = a.colidx + a.rowptr[i + 1];
            const int64_t own = (re - rb) - (std::binary_search(rb, re, (int32_t)i) ? 1 : 0);  // diagonal skipped
            uint32_t *mid = b + own;
            buf.resize((size_t)(e - b));
            uint32_t *o = buf.data();
            uint32_t *x = b, *y = mid;
            while (x < mid || y < e) {
                uint32_t v;
                if (y >= e || (x < mid && *x <= *y)) v = *x++; else v = *y++;
                if (o == buf.data() || o[-1] != v) *o++ = v;
            }
            std::copy(buf.data(), o, b);
            uniq[(size_t)i] = o - buf.data();
        }
    }
    tr.mark("  sort+unique");
    for (int64_t i = 0; i < n; ++i) g.ptr[(size_t)i + 1] = g.ptr[(size_t)i] + uniq[(size_t)i];
    std::vector<int64_t>().swap(indeg);
    g.adj.resize((size_t)g.ptr[(size_t)n]);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; ++i)
        std::copy(tmp.get() + cnt[(size_t)i], tmp.get() + cnt[(size_t)i] + uniq[(size_t)i],
                  g.adj.begin() + g.ptr[(size_t)i]);
    tr.mark("  compact");
    return g;
}

}  // namespace

std::vector<uint32_t> reorder_alg1(const Csr &a)
{
    const int64_t n = a.M;
    if (n > kParallelMinVertices && a.M == a.K) {  // reading R21: the parallel variant at scale
        ParallelReorderParams pp;
        return reorder_alg1_parallel(a, pp);
    }
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


// ============================================================================ reading R21
//
// Alg. 1 at scale (n > kParallelMinVertices, e.g. papers100M-shaped: 111M vertices, 3.2B
// affinity entries): the exact algorithm is sequential in both steps, its dendrogram walk is
// bound by random DRAM accesses (~300 s there) and its ordering costs O(n * L * H).  The
// parallel variant keeps both steps and their rules but relaxes the order of decisions, and
// is a deterministic function of the input and (round, segments, L) -- never of the thread
// count -- so the oracle reproduces it exactly (oracle/reorder.py reorder_parallel):
//   Step I in rounds: the vertices, in ascending (degree, id) order, are cut into rounds of
//   `round` vertices.  Every vertex of a round picks, in parallel and from the state at the
//   round's start, the neighbouring community with the largest merge gain dQ (Eq. 1 as in
//   Q9, ties by smallest id) counting its OWN edges (no edges aggregated from earlier merges);
//   the merges (dQ > 0) are then applied in round order, a target that has meanwhile joined
//   another community being redirected to that community's root (skipped if it is the vertex
//   itself).
//   Step II in segments: the DFS leaf sequence (exact, as in Alg. 1) is cut into `segments`
//   contiguous pieces and the greedy common-neighbour chaining (reading R6) runs in
//   each piece independently (candidates = the next L unvisited vertices of the piece).
ParallelReorderParams::ParallelReorderParams() = default;

std::vector<uint32_t> reorder_alg1_parallel(const Csr &a, const ParallelReorderParams &pp_in)
{
    const int64_t n = a.M;
    std::vector<uint32_t> perm((size_t)n);
    std::iota(perm.begin(), perm.end(), 0u);
    if (n == 0 || a.M != a.K) return perm;
    ParallelReorderParams pp = pp_in;
    if (pp.round <= 0) pp.round = std::max<int64_t>(4096, std::min<int64_t>(1 << 20, n / 4096));
    if (pp.segments <= 0) pp.segments = std::max<int64_t>(1, n / 65536);
    if (pp.L <= 0) pp.L = 8;
    const int H = knobs().reorder_H;
    Trace tr;
    Graph g = affinity_graph(a);
    tr.mark("affinity graph");
    const double m2 = (double)g.ptr[(size_t)n];
    auto deg = [&](int64_t v) { return g.ptr[(size_t)v + 1] - g.ptr[(size_t)v]; };

    // ---- Step I in rounds
    std::vector<uint32_t> parent((size_t)n);
    std::iota(parent.begin(), parent.end(), 0u);
    std::vector<double> acomm((size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v) acomm[(size_t)v] = (double)deg(v);
    // ascending (degree, id): counting sort over the degree values
    std::vector<uint32_t> order((size_t)n);
    {
        int64_t dmax = 0;
        for (int64_t v = 0; v < n; ++v) dmax = std::max<int64_t>(dmax, deg(v));
        std::vector<int64_t> start((size_t)dmax + 2, 0);
        for (int64_t v = 0; v < n; ++v) start[(size_t)deg(v) + 1]++;
        for (int64_t d = 0; d <= dmax; ++d) start[(size_t)d + 1] += start[(size_t)d];
        for (int64_t v = 0; v < n; ++v) order[(size_t)start[(size_t)deg(v)]++] = (uint32_t)v;
    }
    std::vector<uint32_t> first_child((size_t)n, UINT32_MAX), last_child((size_t)n, UINT32_MAX),
        next_sib((size_t)n, UINT32_MAX);
    auto find_ro = [&](uint32_t x) {
        while (parent[x] != x) x = parent[x];
        return x;
    };
    auto find = [&](uint32_t x) {
        uint32_t r = x;
        while (parent[r] != r) r = parent[r];
        while (parent[x] != r) { uint32_t nx = parent[x]; parent[x] = r; x = nx; }
        return r;
    };
    std::vector<uint32_t> proposal((size_t)pp.round), flat;
    int64_t merged_since_flatten = 0;
    double t_decide = 0, t_apply = 0, t_flat = 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](std::chrono::steady_clock::time_point a0, std::chrono::steady_clock::time_point a1) {
        return std::chrono::duration<double, std::milli>(a1 - a0).count();
    };
    for (int64_t r0 = 0; r0 < n; r0 += pp.round) {
        auto t0 = now();
        // parent[] is only a union-find (the merge forest lives in the child lists): flattening
        // it every n/32 merges keeps the read-only root walks of the parallel phase short
        if (merged_since_flatten > n / 32) {
            flat.resize((size_t)n);
#pragma omp parallel for schedule(static)
            for (int64_t v = 0; v < n; ++v) flat[(size_t)v] = find_ro((uint32_t)v);
            parent.swap(flat);
            merged_since_flatten = 0;
        }
        auto t1 = now();
        t_flat += ms(t0, t1);
        const int64_t r1 = std::min<int64_t>(n, r0 + pp.round);
#pragma omp parallel
        {
            std::vector<uint32_t> roots;
#pragma omp for schedule(dynamic, 8)
            for (int64_t i = r0; i < r1; ++i) {
                const uint32_t v = order[(size_t)i];
                uint32_t best = UINT32_MAX;
                const int64_t dv = deg(v);
                if (dv > 0 && m2 > 0.0) {
                    roots.clear();
                    for (int64_t q = g.ptr[v]; q < g.ptr[v + 1]; ++q) {
                        if (q + 16 < g.ptr[v + 1]) __builtin_prefetch(&parent[g.adj[(size_t)q + 16]]);
                        const uint32_t r = find_ro(g.adj[(size_t)q]);
                        if (r != v) roots.push_back(r);
                    }
                    std::sort(roots.begin(), roots.end());
                    double best_dq = 0.0;
                    for (size_t k = 0; k < roots.size();) {
                        size_t e = k;
                        while (e < roots.size() && roots[e] == roots[k]) ++e;
                        const uint32_t r = roots[k];
                        const double dq = 2.0 * ((double)(e - k) / m2 - acomm[r] * acomm[v] / (m2 * m2));
                        if (best == UINT32_MAX || dq > best_dq) { best = r; best_dq = dq; }  // ascending r: ties -> smallest
                        k = e;
                    }
                    if (!(best_dq > 0.0)) best = UINT32_MAX;
                }
                proposal[(size_t)(i - r0)] = best;
            }
        }
        auto t2 = now();
        t_decide += ms(t1, t2);
        for (int64_t i = r0; i < r1; ++i) {
            if (i + 16 < r1) {  // the merges are applied in order: prefetch the targets' state
                const uint32_t rp = proposal[(size_t)(i + 16 - r0)];
                if (rp != UINT32_MAX) {
                    __builtin_prefetch(&parent[rp]);
                    __builtin_prefetch(&acomm[rp], 1);
                    __builtin_prefetch(&last_child[rp]);
                }
                __builtin_prefetch(&acomm[order[(size_t)i + 16]]);
            }
            const uint32_t v = order[(size_t)i];
            const uint32_t r = proposal[(size_t)(i - r0)];
            if (r == UINT32_MAX) continue;
            const uint32_t u = find(r);
            if (u == v) continue;  // the target joined v earlier in this round
            parent[v] = u;
            acomm[u] += acomm[v];
            if (first_child[u] == UINT32_MAX) first_child[u] = v; else next_sib[last_child[u]] = v;
            last_child[u] = v;
            ++merged_since_flatten;
        }
        t_apply += ms(t2, now());
    }
    if (tr.on) std::fprintf(stderr, "[accspmm reorder]   decide %.1f ms, apply %.1f ms, flatten %.1f ms\n", t_decide, t_apply, t_flat);
    tr.mark("step I (dendrogram, rounds)");

    // ---- Step II: DFS leaf sequence (exact), then greedy chaining per segment
    std::vector<uint32_t> seq;
    seq.reserve((size_t)n);
    {
        std::vector<uint32_t> stack, ch;
        for (int64_t r = 0; r < n; ++r) {
            if (parent[(size_t)r] != (uint32_t)r) continue;
            stack.push_back((uint32_t)r);
            while (!stack.empty()) {
                uint32_t x = stack.back();
                stack.pop_back();
                seq.push_back(x);
                ch.clear();
                for (uint32_t c = first_child[x]; c != UINT32_MAX; c = next_sib[c]) ch.push_back(c);
                for (auto it = ch.rbegin(); it != ch.rend(); ++it) stack.push_back(*it);
            }
        }
    }
    // parent[] was path-compressed in Step I; the merge forest lives in the child lists
    std::vector<uint32_t>().swap(parent);
    std::vector<uint32_t>().swap(flat);
    tr.mark("dfs sequence");
    const int64_t nseg = pp.segments, seg = (n + nseg - 1) / nseg;
    const int L = pp.L;
#pragma omp parallel
    {
        // neighbour set of the current source: open addressing with stamps (<= H entries)
        constexpr int kSet = 512;
        std::vector<uint32_t> key(kSet, UINT32_MAX), stampv(kSet, 0);
        uint32_t stamp = 0;
        std::vector<int64_t> nxt, prv;
        std::vector<char> used;
#pragma omp for schedule(dynamic, 1)
        for (int64_t sg = 0; sg < nseg; ++sg) {
            const int64_t s0 = sg * seg, s1 = std::min<int64_t>(n, s0 + seg);
            if (s0 >= s1) continue;
            const int64_t m = s1 - s0;
            nxt.assign((size_t)m + 1, 0);
            prv.assign((size_t)m + 1, 0);
            used.assign((size_t)m, 0);
            for (int64_t i = 0; i <= m; ++i) { nxt[(size_t)i] = i + 1; prv[(size_t)i] = i - 1; }
            nxt[(size_t)m] = 0;
            prv[0] = m;
            prv[(size_t)m] = m - 1;
            nxt[(size_t)m - 1] = m;
            int64_t out = s0;
            auto take = [&](int64_t i) {  // local position i gets the next id
                used[(size_t)i] = 1;
                perm[(size_t)out++] = seq[(size_t)(s0 + i)];
                nxt[(size_t)prv[(size_t)i]] = nxt[(size_t)i];
                prv[(size_t)nxt[(size_t)i]] = prv[(size_t)i];
            };
            for (int64_t i0 = 0; i0 < m; ++i0) {
                if (used[(size_t)i0]) continue;
                take(i0);
                uint32_t v = seq[(size_t)(s0 + i0)];
                while (nxt[(size_t)m] != m) {
                    if (++stamp == 0) { std::fill(stampv.begin(), stampv.end(), 0u); stamp = 1; }
                    const int64_t dv = std::min<int64_t>(H, deg(v));
                    for (int64_t q = 0; q < dv; ++q) {
                        const uint32_t x = g.adj[(size_t)(g.ptr[v] + q)];
                        uint32_t h = (x * 2654435761u) & (kSet - 1);
                        while (stampv[h] == stamp && key[h] != x) h = (h + 1) & (kSet - 1);
                        stampv[h] = stamp;
                        key[h] = x;
                    }
                    int64_t best = -1, best_c = 0;
                    int cand = 0;
                    for (int64_t pi = nxt[(size_t)m]; pi != m && cand < L; pi = nxt[(size_t)pi], ++cand) {
                        const uint32_t u = seq[(size_t)(s0 + pi)];
                        const int64_t du = std::min<int64_t>(H, deg(u));
                        int64_t c = 0;
                        for (int64_t q = 0; q < du; ++q) {
                            const uint32_t x = g.adj[(size_t)(g.ptr[u] + q)];
                            uint32_t h = (x * 2654435761u) & (kSet - 1);
                            while (stampv[h] == stamp && key[h] != x) h = (h + 1) & (kSet - 1);
                            c += stampv[h] == stamp;
                        }
                        if (c > best_c) { best_c = c; best = pi; }
                    }
                    if (best < 0) break;
                    take(best);
                    v = seq[(size_t)(s0 + best)];
                }
            }
        }
    }
    tr.mark("step II (ordering, segments)");
    return perm;
}

}  // namespace accspmm
