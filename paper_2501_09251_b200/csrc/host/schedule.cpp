// Adaptive sparsity-aware load balancing (§3.5) and the
// nnz-balanced multi-GPU partition (BASELINE north_star).
//
// IBD (Eq. 3) decides whether to balance (> 8).  Balanced
// schedules cut the TC-block stream into work units of <= cap blocks
// with near-uniform cost.  Cost per unit follows Eq. (4) with the
// B200 reading of SURVEY Q15: B-row loads scale with the blocks, and the
// write-back of one 8-row window of C costs `wb` block loads (4 B of C vs es_B
// bytes of B per feature: 1 for TF32, 2 for FP16).  Windows longer than the cap
// are split evenly (cross-row write-back); shorter windows are
// concatenated while sum(blocks + wb) <= cap + wb (Fig. 7(b)).
// Unbalanced plans (IBD <= 8 under ACCSPMM_BALANCE_AUTO) may still be `group`ed:
// whole windows concatenated by the same rule, none split (reading R7b: a warp's
// fixed per-unit cost is amortised over short windows).  Grouped plans stop
// concatenating at `group_cap` blocks (reading R7c: min(cap, 32) under the automatic cap):
// long concatenated units cost 1.3-1.9x on the HBM-bound papers100M-shaped matrix.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "../internal.hpp"

namespace accspmm {

double compute_ibd(const std::vector<uint32_t> &rwo)
{
    const size_t W = rwo.size() ? rwo.size() - 1 : 0;
    if (W == 0) return 0.0;
    const double avg = (double)rwo[W] / (double)W;
    double s = 0.0;
    for (size_t w = 0; w < W; ++w) s += std::fabs((double)(rwo[w + 1] - rwo[w]) - avg);
    return s / (double)W;
}

// B200 default: about 192 units per SM (148 SMs; ~12 per resident warp), a multiple
// of 32, in [32, 4096] -- measured on the Reddit-shaped graph.
int auto_cap(int64_t NB)
{
    int64_t c = (NB + 148 * 192 - 1) / (148 * 192);
    c = (c + 31) / 32 * 32;
    return (int)std::max<int64_t>(kPaperCap, std::min<int64_t>(4096, c));
}

int auto_group_cap(int cap)
{
    const int g = knobs().group_cap > 0 ? knobs().group_cap : kGroupCap;  // variants build: sweepable
    return std::max(1, std::min(cap, g));
}

Schedule build_schedule(const std::vector<uint32_t> &rwo, int cap, bool balance, int precision, bool group,
                        int group_cap, int wh)
{
    const int64_t gcap = group_cap > 0 ? group_cap : cap;  // concatenation limit (reading R7c)
    Schedule s;
    s.cap = cap;
    s.balanced = balance;
    s.ibd = compute_ibd(rwo);
    const int64_t W = rwo.size() ? (int64_t)rwo.size() - 1 : 0;
    if (!balance && !group) {
        s.units.reserve((size_t)W);
        for (int64_t w = 0; w < W; ++w)
            s.units.push_back({(uint32_t)w, 1u, rwo[(size_t)w], rwo[(size_t)w + 1], kNoSplit, 0u, 1u, 0u});
        return s;
    }
    // C write-back of one window in TC-block loads: wh rows x N x 4 B over 8 rows x N x es_B
    const int64_t wb = (precision == ACCSPMM_FP16 ? 2 : 1) * (wh / kWindow);
    bool open = false;
    Unit cur{};
    int64_t cost = 0;
    auto close = [&]() {
        if (open) s.units.push_back(cur);
        open = false;
    };
    for (int64_t w = 0; w < W; ++w) {
        const int64_t nb = (int64_t)rwo[(size_t)w + 1] - (int64_t)rwo[(size_t)w];
        if (nb > cap && balance) {
            close();
            const int64_t nseg = (nb + cap - 1) / cap;
            for (int64_t k = 0; k < nseg; ++k) {
                uint32_t b0 = rwo[(size_t)w] + (uint32_t)((k * nb) / nseg);
                uint32_t b1 = rwo[(size_t)w] + (uint32_t)(((k + 1) * nb) / nseg);
                s.units.push_back({(uint32_t)w, 1u, b0, b1, (uint32_t)s.n_split, (uint32_t)k, (uint32_t)nseg,
                                   (uint32_t)(s.n_segments + k)});
            }
            s.n_split += 1;
            s.n_segments += nseg;
        } else {
            const int64_t c = nb + wb;
            if (open && (int64_t)cur.nw < kWmax && cost + c <= gcap + wb) {
                cur.nw += 1;
                cur.b1 = rwo[(size_t)w + 1];
                cost += c;
            } else {
                close();
                cur = {(uint32_t)w, 1u, rwo[(size_t)w], rwo[(size_t)w + 1], kNoSplit, 0u, 1u, 0u};
                cost = c;
                open = true;
            }
        }
    }
    close();
    return s;
}

std::vector<int64_t> partition_bounds(const Csr &a, const std::vector<uint32_t> &perm, int nparts, int wh)
{
    const int64_t W = (a.M + wh - 1) / wh;
    std::vector<int64_t> pre((size_t)W + 1, 0);
    for (int64_t w = 0; w < W; ++w) {
        int64_t s = 0;
        for (int64_t r = w * wh; r < std::min<int64_t>(a.M, (w + 1) * wh); ++r) {
            int64_t o = perm.empty() ? r : (int64_t)perm[(size_t)r];
            s += a.rowptr[o + 1] - a.rowptr[o];
        }
        pre[(size_t)w + 1] = pre[(size_t)w] + s;
    }
    const int64_t nnz = pre[(size_t)W];
    std::vector<int64_t> b((size_t)nparts + 1, 0);
    for (int k = 1; k < nparts; ++k) {
        // b_k = min{ w : nparts * pre(w) >= k * nnz }  (exact integers)
        int64_t lo = 0, hi = W;
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if ((int64_t)nparts * pre[(size_t)mid] >= (int64_t)k * nnz) hi = mid; else lo = mid + 1;
        }
        b[(size_t)k] = lo;
    }
    b[(size_t)nparts] = W;
    return b;
}

}  // namespace accspmm
