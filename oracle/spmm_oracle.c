/*
 * oracle/spmm_oracle.c -- FP64 CSR SpMM oracle and elementwise error bound.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header or constant with paper_2501_09251_b200/ (the
 * product path), and the product path never calls it.
 *
 * Definition followed ("Given an m-by-k
 * sparse matrix A and a k-by-n dense matrix B, SpMM computes A multiply B and
 * obtains an m-by-n dense matrix C"; SPEC.md S:80-88 spmm_oracle):
 *
 *     C[i][j] = sum_{p = rowptr[i]}^{rowptr[i+1]-1}  a[p] * B[colidx[p]][j]
 *     S[i][j] = sum_{p}                            |a[p]| * |B[colidx[p]][j]|
 *
 * The caller passes the already-rounded operands (rho(A), rho(B), see
 * oracle/rounding.py) as float32, which hold TF32/FP16 values exactly.  Every
 * product and sum is IEEE binary64, accumulated sequentially in CSR order, one
 * row per thread, so the result does not depend on the thread count.
 *
 * Pinned by tests/test_oracle_spmm.py: dense numpy float64 GEMM brute force,
 * the SPEC S:86-88 worked examples, and exactness on integer-valued inputs.
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Computes rows `rows[0..nrows)` (or all M rows if rows == NULL) into the
 * row-major outputs C[nrows][N] and S[nrows][N] (S may be NULL).
 * Returns 0 on success, 1 on a dimension / index error. */
int oracle_spmm_fp64(int64_t M, int64_t K,
                     const int64_t *rowptr, const int32_t *colidx, const float *a,
                     const float *B, int64_t N,
                     const int64_t *rows, int64_t nrows,
                     double *C, double *S, int nthreads)
{
    if (M < 0 || K < 0 || N < 0) return 1;
    int64_t R = rows ? nrows : M;
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 64) reduction(| : bad)
    for (int64_t q = 0; q < R; ++q) {
        int64_t i = rows ? rows[q] : q;
        double *c = C + q * N;
        double *s = S ? S + q * N : NULL;
        for (int64_t j = 0; j < N; ++j) { c[j] = 0.0; if (s) s[j] = 0.0; }
        if (i < 0 || i >= M) { bad = 1; continue; }
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
            int64_t k = colidx[p];
            if (k < 0 || k >= K) { bad = 1; break; }
            double av = (double)a[p];
            const float *b = B + k * N;
            for (int64_t j = 0; j < N; ++j) {
                double bv = (double)b[j];
                c[j] += av * bv;
                if (s) s[j] += fabs(av) * fabs(bv);
            }
        }
    }
    return bad;
}

/* Reports the number of OpenMP threads a parallel region would use. */
int oracle_num_threads(int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) return nthreads;
    return omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}
