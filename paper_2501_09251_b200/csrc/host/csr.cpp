// CSR validation and input rounding rho (host side of plan creation, SURVEY §3 call stack step 1-2).
#include <algorithm>
#include <vector>
#include <cstring>

#include "../internal.hpp"

namespace accspmm {

// Canonical CSR (SURVEY §8(b) "Plan validation"): rowptr[0] = 0,
// non-decreasing; columns strictly ascending within a row and in [0, K).
accspmm_status validate_csr(const Csr &a)
{
    if (a.M < 0 || a.K < 0) return fail(ACCSPMM_ERR_INVALID_VALUE, "negative matrix dimension");
    if (a.M == 0) return ACCSPMM_OK;
    if (!a.rowptr) return fail(ACCSPMM_ERR_INVALID_VALUE, "rowptr is NULL");
    if (a.rowptr[0] != 0) return fail(ACCSPMM_ERR_INVALID_CSR, "rowptr[0] != 0");
    const int64_t nnz = a.rowptr[a.M];
    if (nnz < 0) return fail(ACCSPMM_ERR_INVALID_CSR, "rowptr[M] < 0");
    if (nnz > 0 && !a.colidx) return fail(ACCSPMM_ERR_INVALID_VALUE, "colidx is NULL");
    int64_t bad_row = -1;
    int bad_kind = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(max : bad_row, bad_kind)
    for (int64_t i = 0; i < a.M; ++i) {
        int64_t s = a.rowptr[i], e = a.rowptr[i + 1];
        if (e < s || e > nnz) { bad_row = i; bad_kind = 1; continue; }
        for (int64_t p = s; p < e; ++p) {
            int32_t c = a.colidx[p];
            if (c < 0 || c >= a.K) { bad_row = i; bad_kind = 2; break; }
            if (p > s && c <= a.colidx[p - 1]) { bad_row = i; bad_kind = 3; break; }
        }
    }
    if (bad_row >= 0) {
        const char *what = bad_kind == 1 ? "rowptr not monotone" : bad_kind == 2 ? "column index out of range"
                                                                                : "columns not strictly ascending";
        return fail(ACCSPMM_ERR_INVALID_CSR, std::string(what) + " at row " + std::to_string(bad_row));
    }
    return ACCSPMM_OK;
}

// TF32 round-to-nearest, ties away from zero, on the float32 bit pattern
// (SURVEY §8(c) Q1 -- the semantics of PTX cvt.rna.tf32.f32 on sm_100a, which
// truncates NaN payloads instead of rounding them; reading R1).
float round_tf32_rna(float x)
{
    uint32_t u;
    std::memcpy(&u, &x, 4);
    const bool nan = (u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu) != 0u;
    u = nan ? (u & 0xFFFFE000u) : ((u + 0x1000u) & 0xFFFFE000u);
    float y;
    std::memcpy(&y, &u, 4);
    return y;
}

// IEEE binary16, round-to-nearest-even.
uint16_t round_fp16_rne(float x)
{
    _Float16 h = static_cast<_Float16>(x);
    uint16_t b;
    std::memcpy(&b, &h, 2);
    return b;
}

// A^T in canonical CSR (the operand of the backward pass dB = A^T . dC).  Counting sort
// by column; rows are visited in ascending order, so each transposed row comes out sorted.
void csr_transpose(const Csr &a, const float *vals, int64_t *t_rowptr, int32_t *t_colidx, float *t_vals)
{
    const int64_t nnz = a.M ? a.rowptr[a.M] : 0;
    std::fill(t_rowptr, t_rowptr + a.K + 1, 0);
    for (int64_t p = 0; p < nnz; ++p) t_rowptr[a.colidx[p] + 1]++;
    for (int64_t j = 0; j < a.K; ++j) t_rowptr[j + 1] += t_rowptr[j];
    std::vector<int64_t> fill(t_rowptr, t_rowptr + a.K);
    for (int64_t i = 0; i < a.M; ++i)
        for (int64_t p = a.rowptr[i]; p < a.rowptr[i + 1]; ++p) {
            const int64_t q = fill[(size_t)a.colidx[p]]++;
            t_colidx[q] = (int32_t)i;
            if (t_vals) t_vals[q] = vals ? vals[p] : 0.0f;
        }
}

}  // namespace accspmm
