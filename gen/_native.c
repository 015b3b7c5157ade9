/*
 * gen/_native.c -- fast, thread-count-independent helpers for the synthetic
 * input generators (gen/matrices.py).  Input plumbing only: no arithmetic of
 * the SpMM method lives here (no rounding, tiling, encoding or product).
 *
 *  gen_pairs_to_csr : (row, col) pairs -> canonical CSR (sorted, deduplicated),
 *                     optionally symmetrised and with self-loops dropped.
 *  gen_dcsbm_draw   : DC-SBM edge draws with a counter-based RNG (splitmix64),
 *                     so the result does not depend on the number of threads.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static inline double u01(uint64_t seed, uint64_t ctr)
{
    return (double)(splitmix64(seed * 0x100000001B3ull + ctr) >> 11) * (1.0 / 9007199254740992.0);
}

/* first index i in [lo, hi) with a[i] > x, clamped to hi-1 */
static inline int64_t upper(const double *a, int64_t lo, int64_t hi, double x)
{
    int64_t l = lo, h = hi;
    while (l < h) {
        int64_t m = l + ((h - l) >> 1);
        if (a[m] > x) h = m; else l = m + 1;
    }
    return l < hi ? l : hi - 1;
}

void gen_dcsbm_draw(int64_t E, int64_t n, const double *cum, const int32_t *comm,
                    const int64_t *order, const double *cum_sorted, const int64_t *starts,
                    const int64_t *ends, const double *base, const double *tot, double mu,
                    uint64_t seed, int64_t *src, int64_t *dst)
{
    const double total = cum[n - 1];
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        uint64_t c0 = 4ull * (uint64_t)e;
        int64_t s = upper(cum, 0, n, u01(seed, c0) * total);
        int64_t d;
        if (u01(seed, c0 + 1) < mu) {
            d = upper(cum, 0, n, u01(seed, c0 + 2) * total);
        } else {
            int32_t c = comm[s];
            double t = base[c] + u01(seed, c0 + 2) * tot[c];
            int64_t p = upper(cum_sorted, starts[c], ends[c], t);
            d = order[p];
        }
        src[e] = s;
        dst[e] = d;
    }
}

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Returns nnz (>= 0) or -1 on an out-of-range index.  colidx must hold
 * npairs * (symmetric ? 2 : 1) entries; rowptr holds M+1. */
int64_t gen_pairs_to_csr(int64_t npairs, const int64_t *rows, const int64_t *cols, int64_t M,
                         int64_t K, int symmetric, int drop_diag, int64_t *rowptr, int32_t *colidx)
{
    int64_t total = npairs * (symmetric ? 2 : 1);
    int64_t *cnt = (int64_t *)calloc((size_t)M + 1, sizeof(int64_t));
    int bad = 0;
#pragma omp parallel for reduction(| : bad)
    for (int64_t i = 0; i < npairs; ++i) {
        int64_t r = rows[i], c = cols[i];
        if (r < 0 || r >= M || c < 0 || c >= K || (symmetric && (c >= M || r >= K))) { bad = 1; continue; }
        if (drop_diag && r == c) continue;
#pragma omp atomic
        cnt[r + 1]++;
        if (symmetric) {
#pragma omp atomic
            cnt[c + 1]++;
        }
    }
    if (bad) { free(cnt); return -1; }
    for (int64_t i = 0; i < M; ++i) cnt[i + 1] += cnt[i];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ((size_t)M + 1));
    memcpy(fill, cnt, sizeof(int64_t) * ((size_t)M + 1));
    int32_t *tmp = colidx; /* scatter in place, compact afterwards */
    (void)total;
#pragma omp parallel for
    for (int64_t i = 0; i < npairs; ++i) {
        int64_t r = rows[i], c = cols[i];
        if (drop_diag && r == c) continue;
        int64_t p;
#pragma omp atomic capture
        p = fill[r]++;
        tmp[p] = (int32_t)c;
        if (symmetric) {
#pragma omp atomic capture
            p = fill[c]++;
            tmp[p] = (int32_t)r;
        }
    }
    int64_t *uniq = (int64_t *)calloc((size_t)M + 1, sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < M; ++i) {
        int32_t *a = tmp + cnt[i];
        int64_t len = cnt[i + 1] - cnt[i];
        if (len > 1) qsort(a, (size_t)len, sizeof(int32_t), cmp_i32);
        int64_t u = 0;
        for (int64_t j = 0; j < len; ++j)
            if (j == 0 || a[j] != a[j - 1]) a[u++] = a[j];
        uniq[i + 1] = u;
    }
    rowptr[0] = 0;
    for (int64_t i = 0; i < M; ++i) rowptr[i + 1] = rowptr[i] + uniq[i + 1];
    /* compact: rows move only towards lower addresses, so a sequential pass is safe */
    for (int64_t i = 0; i < M; ++i) {
        int64_t len = uniq[i + 1];
        if (rowptr[i] != cnt[i] && len > 0)
            memmove(colidx + rowptr[i], tmp + cnt[i], sizeof(int32_t) * (size_t)len);
    }
    int64_t nnz = rowptr[M];
    free(cnt); free(fill); free(uniq);
    return nnz;
}

/* ------------------------------------------------------------------------
 * Config X (papers100M-shaped): directed graph, out-degree
 * round(lognormal(mu, sigma)) rescaled to mean `mean_deg` and capped at dmax,
 * columns ~ Cat(p) with p_j = 1 + Lomax(alpha) (alias method), deduplicated per
 * row.  Row i's draws use counters derived from (seed, i) only, so the output
 * does not depend on the thread count.
 * ---------------------------------------------------------------------- */
#include <math.h>

static inline double normal01(uint64_t seed, uint64_t ctr)
{
    double u1 = u01(seed, ctr), u2 = u01(seed, ctr + 1);
    if (u1 < 1e-300) u1 = 1e-300;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

void gen_x_degrees(int64_t n, double mean_deg, double mu, double sigma, int64_t dmax, uint64_t seed, int64_t *deg)
{
    const double scale = mean_deg / exp(mu + 0.5 * sigma * sigma);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double x = exp(mu + sigma * normal01(seed, 2ull * (uint64_t)i)) * scale;
        int64_t d = (int64_t)llround(x);
        if (d < 1) d = 1;
        if (d > dmax) d = dmax;
        if (d > n) d = n;
        deg[i] = d;
    }
}

/* Vose alias table over weights w[0..n): prob[], alias[] (caller-allocated). */
void gen_alias_build(int64_t n, const double *w, double *prob, int64_t *alias)
{
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) total += w[i];
    int64_t *small = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *large = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t ns = 0, nl = 0;
    for (int64_t i = 0; i < n; ++i) {
        prob[i] = w[i] * (double)n / total;
        if (prob[i] < 1.0) small[ns++] = i; else large[nl++] = i;
    }
    while (ns > 0 && nl > 0) {
        int64_t s = small[--ns], l = large[--nl];
        alias[s] = l;
        prob[l] = (prob[l] + prob[s]) - 1.0;
        if (prob[l] < 1.0) small[ns++] = l; else large[nl++] = l;
    }
    while (nl > 0) { int64_t l = large[--nl]; prob[l] = 1.0; alias[l] = l; }
    while (ns > 0) { int64_t s = small[--ns]; prob[s] = 1.0; alias[s] = s; }
    free(small);
    free(large);
}

/* Fills row i's draws at colidx[off[i] .. off[i]+deg_i), sorts and deduplicates each
 * row in place; uniq[i] receives the unique count.  Then compacts into CSR:
 * rowptr (n+1) and colidx[0 .. rowptr[n]).  Returns rowptr[n]. */
int64_t gen_x_fill(int64_t n, int64_t ncols, const int64_t *off, const double *prob, const int64_t *alias,
                   uint64_t seed, int32_t *colidx, int64_t *rowptr)
{
    int64_t *uniq = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
        int64_t d = off[i + 1] - off[i];
        int32_t *a = colidx + off[i];
        uint64_t base = 0x5851F42D4C957F2Dull ^ ((uint64_t)i << 20);
        for (int64_t k = 0; k < d; ++k) {
            double u = u01(seed, base + 2ull * (uint64_t)k) * (double)ncols;
            int64_t j = (int64_t)u;
            if (j >= ncols) j = ncols - 1;
            double f = u - (double)j;
            a[k] = (int32_t)(f < prob[j] ? j : alias[j]);
        }
        if (d > 1) qsort(a, (size_t)d, sizeof(int32_t), cmp_i32);
        int64_t u = 0;
        for (int64_t k = 0; k < d; ++k)
            if (k == 0 || a[k] != a[k - 1]) a[u++] = a[k];
        uniq[i] = u;
    }
    rowptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) rowptr[i + 1] = rowptr[i] + uniq[i];
    for (int64_t i = 0; i < n; ++i)
        if (rowptr[i] != off[i] && uniq[i] > 0)
            memmove(colidx + rowptr[i], colidx + off[i], sizeof(int32_t) * (size_t)uniq[i]);
    int64_t nnz = rowptr[n];
    free(uniq);
    return nnz;
}
