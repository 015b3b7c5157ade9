// Hot-column order (reading R22, DESIGN.md §3/§6): the columns of A sorted by descending
// in-degree over the plan's rows (ties by ascending id).  Relabelling the columns in this order
// (c -> its rank) makes every RowWindow condense its most referenced columns first (the paper's
// ascending condensed order, P:257 / SURVEY Q4, applied to the new ids), so the TC blocks of a
// window run from hot to cold and one L2 policy per block (evict_last for the hot set,
// evict_first otherwise) keeps the B rows that many windows gather resident when B exceeds L2.
#include <algorithm>
#include <atomic>
#include <vector>

#include "../internal.hpp"

namespace accspmm {

bool hot_column_order(const Csr &a, const std::vector<uint32_t> &perm, int64_t r0, int64_t r1, bool force,
                      std::vector<uint32_t> &colorig)
{
    const int64_t K = a.K;
    colorig.clear();
    if (K <= 0) return false;
    // in-degree of every column over the plan's (reordered) rows [r0, r1)
    std::vector<uint32_t> deg((size_t)K, 0u);
    int64_t nnz = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : nnz)
    for (int64_t r = r0; r < r1; ++r) {
        const int64_t o = perm.empty() ? r : (int64_t)perm[(size_t)r];
        for (int64_t q = a.rowptr[o]; q < a.rowptr[o + 1]; ++q)
            __atomic_fetch_add(&deg[(size_t)a.colidx[q]], 1u, __ATOMIC_RELAXED);
        nnz += a.rowptr[o + 1] - a.rowptr[o];
    }
    if (nnz == 0) return false;
    // counting sort by descending degree, stable in the column id
    uint32_t dmax = 0;
    for (int64_t c = 0; c < K; ++c) dmax = std::max(dmax, deg[(size_t)c]);
    std::vector<int64_t> start((size_t)dmax + 2, 0);
    for (int64_t c = 0; c < K; ++c) ++start[(size_t)(dmax - deg[(size_t)c]) + 1];
    for (size_t d = 1; d < start.size(); ++d) start[d] += start[d - 1];
    colorig.assign((size_t)K, 0u);
    for (int64_t c = 0; c < K; ++c) colorig[(size_t)start[(size_t)(dmax - deg[(size_t)c])]++] = (uint32_t)c;
    if (!force) {
        // AUTO: only a skewed reference distribution has a hot set worth protecting -- the 1%
        // most referenced of the referenced columns carry >= kHotSkew of the nnz (a uniform
        // distribution gives ~1%)
        int64_t used = 0;
        for (int64_t c = 0; c < K; ++c) used += deg[(size_t)c] > 0;
        const int64_t top = std::max<int64_t>(1, (used + 99) / 100);
        int64_t hot = 0;
        for (int64_t i = 0; i < top; ++i) hot += deg[(size_t)colorig[(size_t)i]];
        if ((double)hot < kHotSkew * (double)nnz) {
            colorig.clear();
            return false;
        }
    }
    return true;
}

}  // namespace accspmm
