// BitTCF format builder (§3.3).
//
// For every RowWindow of 8 consecutive (reordered) rows: the window's non-empty
// columns, ascending (reading SURVEY Q4), are cut into groups of 8 -> one 8x8 TC
// block each.  RowWindowOffset = prefix count of blocks,
// TCOffset = prefix count of nnz, SparseAToB = the original column of
// each condensed lane, 0 for padding (Q5), TCLocalBit = u64 occupancy with
// bit k = r*8 + lane (Q3).  Values are placed at TCOffset[b] + popc(mask & (2^k-1)),
// i.e. ascending bit order inside a block -- the decode rule of P:273 used in
// reverse.  With a column map (symmetric reordering, NEXT-2) columns are relabelled
// c -> colmap[c] before the window's condensed set is formed.  Windows are
// independent, so every pass is an OpenMP loop over windows.
//
// Window height wh (reading R20): wh = 8 is the paper's format.  wh = 16 / 32
// are the tall windows of the tcgen05 path: a window of wh rows is condensed the same way
// into wh x 8 tiles, whose occupancy is wh/8 u64 words per block (word j = tile rows
// 8j..8j+7, bit (r mod 8)*8 + lane inside the word), values in ascending tile position
// r*8 + lane -- the P:273 popcount rule applied to the concatenated words.
#include <algorithm>
#include <cstring>

#include "../internal.hpp"

namespace accspmm {

namespace {

inline int64_t orig_row(const std::vector<uint32_t> &perm, int64_t r)
{
    return perm.empty() ? r : (int64_t)perm[(size_t)r];
}

inline int32_t col_of(const uint32_t *colmap, int32_t c) { return colmap ? (int32_t)colmap[c] : c; }

// sorted unique (relabelled) columns of reordered rows [r0, r1)
inline void window_columns(const Csr &a, const std::vector<uint32_t> &perm, int64_t r0, int64_t r1,
                           std::vector<int32_t> &buf, const uint32_t *colmap = nullptr)
{
    buf.clear();
    for (int64_t r = r0; r < r1; ++r) {
        int64_t o = orig_row(perm, r);
        if (colmap)
            for (int64_t p = a.rowptr[o]; p < a.rowptr[o + 1]; ++p) buf.push_back(col_of(colmap, a.colidx[p]));
        else
            buf.insert(buf.end(), a.colidx + a.rowptr[o], a.colidx + a.rowptr[o + 1]);
    }
    std::sort(buf.begin(), buf.end());
    buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
}

}  // namespace

int64_t count_blocks(const Csr &a, const std::vector<uint32_t> &perm, int wh)
{
    const int64_t W = (a.M + wh - 1) / wh;
    int64_t total = 0;
#pragma omp parallel reduction(+ : total)
    {
        std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 64)
        for (int64_t w = 0; w < W; ++w) {
            window_columns(a, perm, w * wh, std::min<int64_t>(a.M, (w + 1) * wh), buf);
            total += ((int64_t)buf.size() + kWindow - 1) / kWindow;
        }
    }
    return total;
}

accspmm_status build_format(const Csr &a, const float *vals, const std::vector<uint32_t> &perm,
                            int64_t row_begin, int64_t row_end, int precision, HostFormat &out,
                            const uint32_t *colmap, int wh)
{
    const int64_t rows = row_end - row_begin;
    const int64_t W = (rows + wh - 1) / wh;
    const int nw = wh / kWindow;  // u64 occupancy words per block
    out = HostFormat();
    out.rows = rows;
    out.W = W;
    out.wh = wh;
    std::vector<int64_t> U((size_t)W, 0);
    // pass 1: |U_w|
#pragma omp parallel
    {
        std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 64)
        for (int64_t w = 0; w < W; ++w) {
            int64_t r0 = row_begin + w * wh, r1 = std::min(row_end, r0 + wh);
            window_columns(a, perm, r0, r1, buf, colmap);
            U[(size_t)w] = (int64_t)buf.size();
        }
    }
    // RowWindowOffset
    std::vector<int64_t> rwo64((size_t)W + 1, 0);
    for (int64_t w = 0; w < W; ++w) {
        rwo64[(size_t)w + 1] = rwo64[(size_t)w] + (U[(size_t)w] + kWindow - 1) / kWindow;
        out.sum_U += U[(size_t)w];
    }
    const int64_t NB = rwo64[(size_t)W];
    if (NB * kWindow >= (int64_t)UINT32_MAX) return fail(ACCSPMM_ERR_UNSUPPORTED, "8*NB overflows u32 offsets");
    int64_t nnz = 0;
    for (int64_t r = row_begin; r < row_end; ++r) {
        int64_t o = orig_row(perm, r);
        nnz += a.rowptr[o + 1] - a.rowptr[o];
    }
    if (nnz >= (int64_t)UINT32_MAX) return fail(ACCSPMM_ERR_UNSUPPORTED, "plan nnz overflows u32 TCOffset");
    out.NB = NB;
    out.nnz = nnz;
    try {
        out.rwo.resize((size_t)W + 1);
        out.a2b.assign((size_t)NB * kWindow, 0u);
        out.bits.assign((size_t)NB * nw, 0ull);
        out.tco.resize((size_t)NB + 1);
        if (precision == ACCSPMM_FP16) out.v16.resize((size_t)nnz);
        else out.v32.resize((size_t)nnz);
    } catch (...) {
        return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "host allocation of the BitTCF arrays failed");
    }
    for (int64_t w = 0; w <= W; ++w) out.rwo[(size_t)w] = (uint32_t)rwo64[(size_t)w];
    // pass 2: SparseAToB and TCLocalBit
#pragma omp parallel
    {
        std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 64)
        for (int64_t w = 0; w < W; ++w) {
            int64_t r0 = row_begin + w * wh, r1 = std::min(row_end, r0 + wh);
            window_columns(a, perm, r0, r1, buf, colmap);
            const int64_t base = rwo64[(size_t)w];
            for (size_t q = 0; q < buf.size(); ++q) out.a2b[(size_t)base * kWindow + q] = (uint32_t)buf[q];
            for (int64_t r = r0; r < r1; ++r) {
                int64_t o = orig_row(perm, r);
                const int lr = (int)(r - r0);
                for (int64_t p = a.rowptr[o]; p < a.rowptr[o + 1]; ++p) {
                    size_t pos = (size_t)(std::lower_bound(buf.begin(), buf.end(), col_of(colmap, a.colidx[p])) - buf.begin());
                    out.bits[((size_t)base + pos / kWindow) * nw + lr / kWindow] |=
                        1ull << ((lr % kWindow) * kWindow + (int)(pos % kWindow));
                }
            }
        }
    }
    // TCOffset = popcount prefix sums (all words of a block)
    out.tco[0] = 0;
    for (int64_t b = 0; b < NB; ++b) {
        uint32_t c = 0;
        for (int j = 0; j < nw; ++j) c += (uint32_t)__builtin_popcountll(out.bits[(size_t)b * nw + j]);
        out.tco[(size_t)b + 1] = out.tco[(size_t)b] + c;
    }
    // pass 3: values, rounded with rho and placed by the popcount rule of P:273
#pragma omp parallel
    {
        std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 64)
        for (int64_t w = 0; w < W; ++w) {
            int64_t r0 = row_begin + w * wh, r1 = std::min(row_end, r0 + wh);
            window_columns(a, perm, r0, r1, buf, colmap);
            const int64_t base = rwo64[(size_t)w];
            for (int64_t r = r0; r < r1; ++r) {
                int64_t o = orig_row(perm, r);
                const int lr = (int)(r - r0);
                for (int64_t p = a.rowptr[o]; p < a.rowptr[o + 1]; ++p) {
                    size_t pos = (size_t)(std::lower_bound(buf.begin(), buf.end(), col_of(colmap, a.colidx[p])) - buf.begin());
                    size_t b = (size_t)base + pos / kWindow;
                    const int word = lr / kWindow;
                    int k = (lr % kWindow) * kWindow + (int)(pos % kWindow);
                    size_t idx = out.tco[b];
                    for (int j = 0; j < word; ++j) idx += (size_t)__builtin_popcountll(out.bits[b * nw + j]);
                    uint64_t below = out.bits[b * nw + word] & ((1ull << k) - 1ull);
                    idx += (size_t)__builtin_popcountll(below);
                    float v = vals ? vals[p] : 0.0f;
                    if (precision == ACCSPMM_FP16) out.v16[idx] = round_fp16_rne(v);
                    else out.v32[idx] = round_tf32_rna(v);
                }
            }
        }
    }
    return ACCSPMM_OK;
}

}  // namespace accspmm
