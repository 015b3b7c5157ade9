/*
 * accspmm.h -- C ABI of the B200-native Acc-SpMM hot path (arXiv 2501.09251).
 *
 * Operation (§5): "Given an m-by-k sparse matrix A and a
 * k-by-n dense matrix B, SpMM computes A multiply B and obtains an m-by-n dense
 * matrix C."  A is held in the paper's BitTCF format (§3.3): RowWindows
 * of 8 rows whose non-empty columns are condensed into 8x8 TC blocks, each with a
 * uint64 occupancy bitmap.  Work is balanced over SMs by the
 * sparsity-aware scheduler of §3.5.  Inputs are rounded once with
 * rho = TF32 round-to-nearest-away ("tf32"; reading SURVEY §8(c) Q1) or
 * FP16 round-to-nearest-even (BASELINE north_star "plus an FP16 variant"), and
 * products accumulate in FP32.
 *
 * Conventions (all functions):
 *   - Sparse A is canonical CSR on the HOST: rowptr int64[M+1] (rowptr[0] = 0,
 *     non-decreasing), colidx int32[nnz] strictly ascending within each row and
 *     in [0, K), vals float32[nnz].  The arrays are borrowed for the duration of
 *     plan creation only; the caller may free them afterwards.
 *   - Dense B is K x N row-major, contiguous (leading dimension N), on the
 *     plan's device: float32 for ACCSPMM_TF32, IEEE binary16 for ACCSPMM_FP16;
 *     16-byte aligned.  C is float32, row-major, leading dimension N, 16-byte
 *     aligned, caller-owned, on the plan's device.
 *   - N >= 1.  The kernels run on feature widths Np = 16, 32, 64 or a multiple of
 *     128; any other N goes through a zero-padded K x Np copy of B and a padded C
 *     (two 2-D copies on the stream, plan-owned scratch; Np = the next such width),
 *     so any N and any alignment of B and C is accepted there.
 *   - Streams are CUDA runtime streams passed as `void*` (cudaStream_t); NULL
 *     is the legacy default stream.
 *   - Every function returns a status; on failure a thread-local message is
 *     available from accspmm_last_error().  No function calls exit/abort.
 *   - There is no CPU fallback: a plan created for a device executes only with
 *     the CUDA kernels of this library; a host-only plan (device = -1) can be
 *     inspected (info, export) but refuses to execute.
 */
#ifndef ACCSPMM_H
#define ACCSPMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACCSPMM_ABI_VERSION 1

typedef struct accspmm_plan accspmm_plan; /* opaque */

typedef enum {
    ACCSPMM_OK = 0,
    ACCSPMM_ERR_INVALID_VALUE = 1,  /* null pointer, bad size, bad option, misaligned pointer     */
    ACCSPMM_ERR_INVALID_CSR = 2,    /* rowptr not monotone / colidx unsorted, duplicate, out of range */
    ACCSPMM_ERR_UNSUPPORTED = 3,    /* u32 offset overflow, host-only plan, fused all-gather N % 16 */
    ACCSPMM_ERR_OUT_OF_MEMORY = 4,  /* host or device allocation failed                           */
    ACCSPMM_ERR_CUDA = 5,           /* a CUDA runtime call or kernel launch failed                 */
    ACCSPMM_ERR_INTERNAL = 6
} accspmm_status;

typedef enum { ACCSPMM_TF32 = 0, ACCSPMM_FP16 = 1 } accspmm_precision;

typedef enum {
    ACCSPMM_REORDER_OFF = 0,
    ACCSPMM_REORDER_ON = 1,   /* Algorithm 1, rows only (reading SURVEY Q12)      */
    ACCSPMM_REORDER_AUTO = 2  /* keep the permutation only if it reduces the TC-block count   */
} accspmm_reorder_mode;

typedef enum {
    ACCSPMM_BALANCE_OFF = 0,  /* one work unit per RowWindow ("each TB processes all the TC blocks of a single RowWindow") */
    ACCSPMM_BALANCE_ON = 1,   /* TC blocks redistributed into units of <= unit_cap blocks   */
    ACCSPMM_BALANCE_AUTO = 2  /* balance iff IBD (Eq. 3) > 8; otherwise windows stay whole but
                                 consecutive ones are grouped into one warp's unit (B200)        */
} accspmm_balance_mode;

typedef enum {
    ACCSPMM_BUILD_HOST = 0,   /* BitTCF built by the host builder (OpenMP over RowWindows), then uploaded */
    ACCSPMM_BUILD_DEVICE = 1  /* CSR uploaded, BitTCF built by data-parallel device passes (sort + scans);
                                 bit-identical arrays; needs device >= 0                             */
} accspmm_build_mode;

typedef struct {
    int32_t precision;  /* accspmm_precision; default ACCSPMM_TF32                                   */
    int32_t reorder;    /* accspmm_reorder_mode; default ACCSPMM_REORDER_AUTO         */
    int32_t balance;    /* accspmm_balance_mode; default ACCSPMM_BALANCE_AUTO                        */
    int32_t unit_cap;   /* max TC blocks per work unit; 0 = automatic (>= 32, the P:446 threshold)   */
    int32_t part;       /* this rank's part in [0, nparts)                                          */
    int32_t nparts;     /* number of nnz-balanced RowWindow ranges (multi-GPU); 1 = whole matrix    */
    int32_t device;     /* CUDA device ordinal; -1 = host-only plan (format + schedule, no upload)  */
    int32_t build;      /* accspmm_build_mode; default ACCSPMM_BUILD_HOST                            */
    int32_t permute_cols; /* 1: when a row permutation is applied (square A), relabel the columns with
                             it too (A' = P A P^T): windows condense their columns
                             in the new order; the device copy of SparseAToB keeps each column's
                             ORIGINAL id, so execute gathers B's rows directly (no B' = P B
                             pass).  C is unchanged.  Default 0 (rows only, reading Q12).          */
    int32_t window_rows;  /* rows per RowWindow: 0 or 8 = the paper's BitTCF (8x8 tiles);
                             16 or 32 = tall windows (reading R20: wh x 8 tiles, wh/8 u64 occupancy
                             words per block), executed by the tcgen05 kernel (TF32 only) unless
                             kernel = MMA_SYNC, which runs 16-row windows (TF32 or FP16; two
                             accumulator halves per gathered row) and rejects 32.                 */
    int32_t kernel;       /* accspmm_kernel: which SpMM kernel executes the plan (default AUTO)   */
    int32_t hot_cols;     /* accspmm_hot_mode; reading R22 (DESIGN.md §3/§6): relabel the columns by
                             descending in-degree so each window condenses its hottest columns
                             first, and tag every TC block with the hotness of its first column;
                             when B exceeds L2 the kernel then gathers hot blocks with an L2
                             evict_last policy and the rest evict_first.  C is unchanged.  Only
                             for 8-row windows on the mma.sync kernel, without permute_cols, and
                             K < 2^27.  Default AUTO: on iff K >= 2^20 and the 1% most referenced
                             of the referenced columns carry >= 10% of the plan's nnz.            */
    int32_t reserved[4];
} accspmm_options;

typedef enum {
    ACCSPMM_HOT_AUTO = 0,
    ACCSPMM_HOT_ON = 1,
    ACCSPMM_HOT_OFF = 2
} accspmm_hot_mode;

typedef enum {
    ACCSPMM_KERNEL_AUTO = 0,     /* 8-row windows: mma.sync kernel; tall windows: tcgen05 kernel        */
    ACCSPMM_KERNEL_MMA_SYNC = 1, /* TMA gather4 + warp-level mma.sync (8-row windows only)              */
    ACCSPMM_KERNEL_TCGEN05 = 2   /* TMA gather4 + tcgen05.mma with the gathered rows in TMEM, FP32
                                    accumulators in TMEM (TF32; any window height; N % 128 == 0 natively,
                                    other N through the padded path)                                  */
} accspmm_kernel;

typedef struct {
    int64_t M, K, nnz;          /* the input matrix                                                 */
    int64_t rows;               /* rows this plan writes (= M when nparts == 1)                     */
    int64_t row_begin;          /* first (reordered) row of this plan's slab                        */
    int64_t window_begin;       /* first RowWindow of the slab (global index)                       */
    int64_t W, NB;              /* RowWindows and TC blocks in this plan                            */
    int64_t plan_nnz;           /* nnz held by this plan                                            */
    int64_t sum_U;              /* sum over windows of unique columns = B rows gathered (bytes model) */
    int64_t n_units, n_split_windows, n_segments;
    int64_t nb_unreordered;     /* TC blocks of the matrix without reordering (AUTO decision)        */
    int32_t precision, reorder_applied, balanced, unit_cap, perm_present, part, nparts, device;
    double mean_nnz_tc;         /* plan_nnz / NB                                             */
    double ibd;                 /* Eq. (3) over this plan's windows                                  */
    int64_t index_bytes;        /* (ceil(rows/8) + 11*NB + 2)*4                               */
    int64_t metcf_index_bytes;  /* ME-TCF equivalent                                     */
    int64_t csr_index_bytes;    /* (rows+1)*4 + nnz*4                                                */
    int64_t value_bytes;        /* es_A * plan_nnz                                                   */
    int64_t device_bytes;       /* bytes resident on the device for this plan (excl. workspace)      */
    double ms_validate, ms_reorder, ms_build, ms_schedule, ms_upload;
    int64_t grouped;            /* 1: unbalanced plan whose whole windows are grouped per unit (AUTO) */
    int64_t cols_permuted;      /* 1: columns relabelled with the row permutation (permute_cols)      */
    int64_t group_cap;          /* concatenation limit of short windows (blocks): min(cap, 32) for grouped
                                   plans under the automatic cap, else = unit_cap                    */
    int64_t window_rows;        /* rows per RowWindow of this plan (8 = the paper's BitTCF)           */
    int64_t kernel;             /* accspmm_kernel the plan executes with (resolved, never AUTO)       */
    int64_t hot_cols;           /* 1: columns relabelled by in-degree with per-block hotness tags (R22) */
    int64_t reserved[2];
} accspmm_plan_info;

/* Fills *opt with the defaults listed above.  Never fails for a non-null opt. */
accspmm_status accspmm_options_default(accspmm_options *opt);

/* Builds a plan with default options on the current CUDA device.
 * Steps (all host-side, timed into accspmm_plan_info): validate CSR, round vals
 * with rho, optional Algorithm-1 reordering, BitTCF build, IBD +
 * schedule (Eq. 3/4), device upload.  *out receives a plan owned by the caller
 * (free with accspmm_plan_destroy).  M = 0 or nnz = 0 are valid.
 * Errors: INVALID_VALUE (null out, negative sizes, null arrays with nnz > 0),
 * INVALID_CSR, UNSUPPORTED (a u32 offset would overflow), OUT_OF_MEMORY, CUDA. */
accspmm_status accspmm_plan_create(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                   const float *vals, accspmm_plan **out);

/* As accspmm_plan_create with explicit options (opt may be NULL = defaults).
 * With nparts > 1 the plan covers only RowWindows [b_part, b_part+1) of the
 * nnz-balanced partition b_k = min{w : nparts*pre(w) >= k*nnz} (pre = nnz of
 * windows before w, in reordered order). */
accspmm_status accspmm_plan_create_ex(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                      const float *vals, const accspmm_options *opt, accspmm_plan **out);

/* As accspmm_plan_create_ex, with the Algorithm-1 permutation supplied by the caller instead
 * of computed (perm_new2old u32[M], a bijection of [0, M), e.g. the output of accspmm_reorder
 * or accspmm_reorder_parallel computed once and broadcast to every rank of a multi-GPU job).
 * opt->reorder still decides: OFF ignores it, ON applies it, AUTO applies it iff it reduces
 * the TC-block count.  Errors as accspmm_plan_create_ex, plus INVALID_VALUE for a NULL perm,
 * a non-bijection or a non-square A. */
accspmm_status accspmm_plan_create_perm(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                        const float *vals, const accspmm_options *opt,
                                        const uint32_t *perm_new2old, accspmm_plan **out);

/* C = A . B on `stream`, asynchronously (never synchronises the host).
 * nparts == 1: C is M x N in ORIGINAL row order (reordered rows are scattered
 * back through the permutation).  nparts > 1: C is the slab, info.rows x N, in
 * reordered row order (accspmm_plan_export_rows gives each slab row's original id).
 * Every element of C is written (empty rows get 0); there is no beta.
 * B and C are device pointers (see conventions).  The call launches the SpMM
 * kernel, preceded by one pass over B into a plan-owned K x N scratch when
 * (a) the plan is TF32 and every B row is gathered >= 32 times on average
 * (sum_w |U_w| >= 32 K): rho(B) once instead of in the kernel, or (b) the plan
 * has permute_cols: the row gather B' = P B (fused with (a)).  The first call
 * for a given N may allocate the scratch and a split-window workspace
 * (cudaMalloc); later calls only launch kernels on `stream`, so they can be
 * captured into a CUDA graph.  Concurrent executes of one plan on different
 * streams are not allowed (they share the workspace).
 * Errors: INVALID_VALUE (null pointers, N <= 0, B or C not 16-byte aligned when
 * N % 16 == 0), UNSUPPORTED (host-only plan), OUT_OF_MEMORY, CUDA (launch failure). */
accspmm_status accspmm_execute(const accspmm_plan *plan, const void *B, int64_t N, void *C, void *stream);

/* Fused all-gather (multi-GPU, BASELINE "optional all-gather" of the C slabs): instead of
 * writing this plan's slab, the SpMM epilogue writes every finished row, in ORIGINAL row
 * order, into each of the n_dst full M x N float32 matrices C_all[0..n_dst) (1 <= n_dst <= 8;
 * typically this GPU's C and its peers' C mapped through CUDA IPC / symmetric memory over
 * NVLink, which must be accessible from the plan's device).  The gather thus overlaps the
 * compute window by window and needs neither a collective nor the un-permute kernel; after
 * every rank's call completed (a barrier across the ranks' streams, the caller's job) each
 * C_all matrix holds the whole product.  Works for any plan (nparts = 1: all rows).  Errors
 * as accspmm_execute, plus INVALID_VALUE for n_dst out of range or NULL/misaligned entries. */
accspmm_status accspmm_execute_allgather(const accspmm_plan *plan, const void *B, int64_t N, void *const *C_all,
                                         int32_t n_dst, void *stream);

/* End-to-end variant with HOST buffers: copies B (K x N, host) to the device,
 * executes, copies C (host, same shape as accspmm_execute's C) back and
 * synchronises `stream`.  Pinned host memory gives full PCIe bandwidth. */
accspmm_status accspmm_execute_host(const accspmm_plan *plan, const void *B_host, int64_t N, void *C_host,
                                    void *stream);

/* Pipelined end-to-end batch: for i < count, C_hosts[i] = A . B_hosts[i] (shapes and
 * types as accspmm_execute_host).  Two device staging slots and two copy streams
 * overlap the H2D copy of B_{i+1} and the D2H copy of C_{i-1} with the SpMM of step i
 * (PCIe is full duplex), so the steady-state step costs max(H2D, SpMM, D2H) instead of
 * their sum.  Host buffers must be pinned for the copies to overlap (pageable memory is
 * still correct, only serialised).  The SpMM runs on `stream`; returns after every C_i
 * has landed (synchronises).  Errors as accspmm_execute_host. */
accspmm_status accspmm_execute_host_batch(const accspmm_plan *plan, const void *const *B_hosts, void *const *C_hosts,
                                          int32_t count, int64_t N, void *stream);

/* Frees every host and device resource of the plan.  NULL is a no-op.  The
 * caller must ensure no execute on this plan is still in flight. */
void accspmm_plan_destroy(accspmm_plan *plan);

/* Copies plan statistics into *info. */
accspmm_status accspmm_plan_get_info(const accspmm_plan *plan, accspmm_plan_info *info);

/* Bytes per element of B as an execute at width N gathers it (SURVEY §8(d)'s es_B, the
 * per-valid-lane B bytes of the bytes model): 2 for FP16; for TF32 3 when the pre-rounded
 * B is stored as its 3-byte image (B3: bits 31..8 of rho(b), lossless because
 * rho -- P:308, SURVEY Q1 -- leaves bits 12..0 zero; used when the plan's B rows are reused
 * >= 32 times and the feature slice is 64 or 128 wide), else 4.  Host-only, no device work.
 * INVALID_VALUE on NULL arguments or N <= 0. */
accspmm_status accspmm_plan_b_bytes(const accspmm_plan *plan, int64_t N, int32_t *bytes_per_element);

/* Copies the plan's BitTCF arrays to HOST buffers sized from accspmm_plan_info:
 * rwo u32[W+1], tco u32[NB+1], a2b u32[8*NB], bits u64[NB * window_rows/8] (window_rows/8
 * words per block; one for the paper's 8-row windows), vals (float32[plan_nnz]
 * for TF32, uint16 bit patterns for FP16).  Any pointer may be NULL (skipped).
 * Window/block offsets are relative to this plan's slab.  Blocks the host thread. */
accspmm_status accspmm_plan_export_format(const accspmm_plan *plan, uint32_t *rwo, uint32_t *tco, uint32_t *a2b,
                                          uint64_t *bits, void *vals);

/* Copies the n_units work units as u32[n_units][8] = {w0, nw, b0, b1, split_id
 * (0xFFFFFFFF = whole windows), seg, nseg, workspace slot}. */
accspmm_status accspmm_plan_export_units(const accspmm_plan *plan, uint32_t *units);

/* Copies, for each of the plan's info.rows rows, its ORIGINAL row index
 * (u32[rows]); identity when no reordering was applied. */
accspmm_status accspmm_plan_export_rows(const accspmm_plan *plan, uint32_t *orig_row);

/* Algorithm 1 alone (host): perm_new2old u32[n] for the square n x n CSR.
 * Returns INVALID_CSR / INVALID_VALUE as plan creation does. */
accspmm_status accspmm_reorder(int64_t n, const int64_t *rowptr, const int32_t *colidx, uint32_t *perm_new2old);

/* The deterministic parallel variant of Algorithm 1 (host; reading R21), which
 * plan creation uses for graphs above 8M vertices: Step I in rounds of `round` vertices (in
 * ascending degree), every vertex of a round choosing its merge target from the state at the
 * round's start by its own edges, merges applied in round order; Step II's greedy chaining run
 * independently on `segments` contiguous pieces of the DFS sequence with an L-candidate window.
 * round, segments, L <= 0 select the defaults (max(4096, min(2^20, n/4096)), max(1, n/65536),
 * 8).  The result depends only on the input and these parameters (not on the thread count).
 * Errors as accspmm_reorder. */
accspmm_status accspmm_reorder_parallel(int64_t n, const int64_t *rowptr, const int32_t *colidx, int64_t round,
                                        int64_t segments, int32_t L, uint32_t *perm_new2old);

/* A^T (host): the K x M transpose of the canonical CSR A as canonical CSR -- the operand
 * of the backward pass dB = A^T . dC of C = A . B.  t_rowptr int64[K+1], t_colidx
 * int32[nnz], t_vals float32[nnz] (t_vals and vals may be NULL: pattern only), caller-owned.
 * Errors: INVALID_VALUE, INVALID_CSR (as plan creation), UNSUPPORTED (M >= 2^31). */
accspmm_status accspmm_csr_transpose(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                    const float *vals, int64_t *t_rowptr, int32_t *t_colidx, float *t_vals);

/* nnz-balanced partition bounds (host): bounds int64[nparts+1] over the
 * ceil(M/8) 8-row windows of the given CSR (already in the order to be partitioned). */
accspmm_status accspmm_partition_bounds(int64_t M, const int64_t *rowptr, int32_t nparts, int64_t *bounds);

/* Kernel timing (measurement hook).  While enabled, every execute records CUDA
 * events on its stream around the SpMM kernel launch only (not the B rounding
 * pass).  accspmm_plan_kernel_times synchronises on the recorded events, writes
 * up to max_n elapsed times in ms (oldest first) and clears the record; *n_out
 * receives the number written.  At most 4096 launches are kept. */
accspmm_status accspmm_plan_set_timing(accspmm_plan *plan, int32_t enable);
accspmm_status accspmm_plan_kernel_times(accspmm_plan *plan, float *ms_out, int32_t max_n, int32_t *n_out);

/* Multi-GPU helper (device): C[orig_row[i]][:] = G[i][:] for i < n_rows where
 * orig_row[i] != 0xFFFFFFFF (padding of an all-gathered slab set).  G and C are
 * float32 row-major with leading dimension N (multiple of 4). */
accspmm_status accspmm_unpermute(const float *G, const uint32_t *orig_row, int64_t n_rows, int64_t N, float *C,
                                 void *stream);

/* Test hooks (device).  accspmm_debug_round_tf32: out[i] = cvt.rna.tf32.f32(in[i])
 * -- the instruction the kernel applies to B.  accspmm_debug_decode: tiles
 * float32[NB][8*wh] (wh = window_rows), tile[b][r*8+c] = value of (row r, lane c) of TC
 * block b or 0, decoded on the device with the kernel's popcount rule. */
accspmm_status accspmm_debug_round_tf32(const float *in, float *out, int64_t n, void *stream);
accspmm_status accspmm_debug_decode(const accspmm_plan *plan, float *tiles, void *stream);

/* Measurement hook (device, synchronous): L2 read bandwidth of the current device in
 * GB/s.  Allocates an L2-resident buffer of `bytes` (>= 1 MiB; well under the 126 MB L2),
 * warms it, then times `iters` full passes of 128-bit L2-only loads (ld.global.cg) by all
 * SMs with CUDA events.  The SpMM kernel's B-row gathers are served from L2 on graphs
 * whose B fits there, so this is the roofline denominator of its L2 bytes (bench.py). */
accspmm_status accspmm_probe_l2_bandwidth(int64_t bytes, int32_t iters, double *gbs);

/* The same probe with a choice of request engine (device, synchronous): mode 1 = the 128-bit
 * ld.global.cg loads above; mode 2 = TMA bulk copies (cp.async.bulk global -> shared, one
 * issuing thread per CTA, 2-16 KB chunks through a 4-8 stage mbarrier ring: the path the
 * SpMM kernel's gathered B rows take); mode 0 = the larger of the two.  `bytes` is rounded
 * down to a multiple of 16 KiB.  Errors: ACCSPMM_ERR_INVALID_VALUE for bytes < 1 MiB,
 * iters < 1, a NULL gbs or another mode; ACCSPMM_ERR_CUDA for a failed allocation/launch. */
accspmm_status accspmm_probe_l2_bandwidth_ex(int64_t bytes, int32_t iters, int32_t mode, double *gbs);

const char *accspmm_status_string(accspmm_status s);
const char *accspmm_last_error(void);
int32_t accspmm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ACCSPMM_H */
