// Internal declarations shared by the host (C++) and device (CUDA) halves of libaccspmm.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "accspmm.h"

namespace accspmm {

constexpr int kWindow = 8;            // P:250 "8 x 8" TC blocks, P:251 ceil(M/8) windows
constexpr uint32_t kNoSplit = 0xFFFFFFFFu;
constexpr uint32_t kPadLane = 0xFFFFFFFFu;  // device SparseAToB padding lane (row -1: TMA zero fill)
constexpr int kWmax = 31;             // windows per concatenated unit (one per lane of the window table)
constexpr double kIbdThreshold = 8.0; // P:417 "When IBD exceeds 8"
constexpr int kPaperCap = 32;         // P:446 "maximum threshold of 32 TC blocks per TB"
constexpr int kMaxGatherDst = 8;      // destinations of the fused all-gather epilogue (one per GPU)
constexpr int kGroupCap = 32;         // concatenation limit of grouped plans, automatic cap (reading R7c)
// TF32 rho(B): a separate rounding pass over B when every B row is gathered at least this
// many times on average (sum_w |U_w| >= kRoundReuse * K), else cvt.rna in the kernel
constexpr int64_t kRoundReuse = 32;
// Hot columns (reading R22): a block's hotness tag sits in bits 31..27 of its lane-0 device
// SparseAToB entry (column ids < 2^27); the hot set of an execute is the 2^hot_lim hottest
// columns with 2^hot_lim * N * es <= kHotBytes, used only when B exceeds kHotL2Bytes.
constexpr int kHotShift = 27;
constexpr uint32_t kHotIdMask = (1u << kHotShift) - 1u;
constexpr int64_t kHotMinCols = 1 << 20;          // AUTO: K >= 2^20 ...
constexpr double kHotSkew = 0.10;                 // ... and the top 1% of the referenced columns carry >= 10% of nnz
constexpr int64_t kHotBytes = 64ll << 20;         // hot set of one execute (bytes of B)
constexpr int64_t kHotL2Bytes = 96ll << 20;       // B larger than this: hot/cold policies

// Error plumbing (thread-local message returned by accspmm_last_error).
accspmm_status fail(accspmm_status s, const std::string &msg);

// Measurement knobs for A/B sweeps (tools/sweep.py).  Only the variants build
// (-DACCSPMM_VARIANTS -> libaccspmm_variants.so) reads them from ACCSPMM_* environment
// variables; the product library (libaccspmm.so) never calls getenv and always uses these
// defaults, which are the measured choices of DESIGN.md §7.
struct Knobs {
    int kcfg = -1;             // ACCSPMM_KCFG: kernel variant (-1 = default kernel)
    int fw = 0;                // ACCSPMM_FW: feature-slice width override (0 = pick_fw rule)
    int slice_major = 1;       // ACCSPMM_SLICE_MAJOR: slice-major grid when N spans several slices
    int l2promo = 3;           // ACCSPMM_L2PROMO: TMA L2 sector promotion 0..3 = none/64/128/256 B
    int round_b = 0;           // ACCSPMM_ROUND_B: 1 = rho(B) pre-pass, 2 = in-kernel, 0 = reuse rule
    int64_t l2_persist_mib = 0;  // ACCSPMM_L2_PERSIST: L2 persisting window over B (MiB)
    int group_cap = 0;         // ACCSPMM_GROUP_CAP: grouped-plan concatenation limit (0 = kGroupCap)
    int reorder_L = 64;        // ACCSPMM_REORDER_L: Alg. 1 candidate window (reading R6)
    int reorder_H = 128;       // ACCSPMM_REORDER_H: Alg. 1 neighbour-list cap (reading R6)
    int b3 = 0;                // ACCSPMM_B3: 3-byte TF32 image of a pre-rounded B (measured, not taken)
    int64_t hot_bytes = kHotBytes;       // ACCSPMM_HOT_MB: hot-set size of an execute (R22)
    int64_t hot_l2_bytes = kHotL2Bytes;  // ACCSPMM_HOT_L2_MB: B size above which hot/cold policies apply
};
const Knobs &knobs();          // variants build: re-read on every call (sweeps flip them)
constexpr bool kVariantsBuild =
#ifdef ACCSPMM_VARIANTS
    true;
#else
    false;
#endif

struct Csr {
    int64_t M = 0, K = 0;
    const int64_t *rowptr = nullptr;
    const int32_t *colidx = nullptr;
};

// Host-side BitTCF of one plan (a contiguous range of RowWindows of the
// reordered matrix); offsets relative to the slab.
struct HostFormat {
    int64_t W = 0, NB = 0, nnz = 0, rows = 0, sum_U = 0;
    int wh = kWindow;            // rows per RowWindow (8 = the paper's; 16/32 tall windows, R20)
    std::vector<uint32_t> rwo;   // RowWindowOffset u32[W+1]
    std::vector<uint32_t> tco;   // TCOffset        u32[NB+1]
    std::vector<uint32_t> a2b;   // SparseAToB      u32[8 NB]
    std::vector<uint64_t> bits;  // TCLocalBit      u64[NB * wh/8] (wh/8 words per block)
    std::vector<float> v32;      // values (TF32-rounded) when precision == TF32
    std::vector<uint16_t> v16;   // values (FP16 bits) when precision == FP16
};

struct Unit { uint32_t w0, nw, b0, b1, split, seg, nseg, slot; };

struct Schedule {
    std::vector<Unit> units;
    int64_t n_split = 0, n_segments = 0;
    int cap = 0;
    bool balanced = false;
    double ibd = 0.0;
};

// host/csr.cpp
accspmm_status validate_csr(const Csr &a);
float round_tf32_rna(float x);        // (bits + 0x1000) & 0xFFFFE000
uint16_t round_fp16_rne(float x);     // IEEE binary16, ties to even
void csr_transpose(const Csr &a, const float *vals, int64_t *t_rowptr, int32_t *t_colidx, float *t_vals);

// host/bittcf.cpp -- rows [row_begin, row_end) of the row-permuted matrix
// (perm new->old may be empty = identity); row_begin is a multiple of 8.
// colmap (may be null): column relabelling old -> new (the inverse row permutation when
// columns are reordered with the rows, accspmm_options.permute_cols)
accspmm_status build_format(const Csr &a, const float *vals, const std::vector<uint32_t> &perm,
                            int64_t row_begin, int64_t row_end, int precision, HostFormat &out,
                            const uint32_t *colmap = nullptr, int wh = kWindow);
int64_t count_blocks(const Csr &a, const std::vector<uint32_t> &perm, int wh = kWindow);

// host/schedule.cpp
double compute_ibd(const std::vector<uint32_t> &rwo);
int auto_cap(int64_t NB);
Schedule build_schedule(const std::vector<uint32_t> &rwo, int cap, bool balance, int precision, bool group,
                        int group_cap = 0, int wh = kWindow);
int auto_group_cap(int cap);  // concatenation limit under the automatic cap (reading R7c)

// host/partition.cpp
std::vector<int64_t> partition_bounds(const Csr &a, const std::vector<uint32_t> &perm, int nparts,
                                      int wh = kWindow);

// host/reorder.cpp -- Algorithm 1; returns perm new->old (identity for an edgeless graph).
// Above kParallelMinVertices the deterministic parallel variant of reading R21 runs instead.
constexpr int64_t kParallelMinVertices = 8'000'000;
struct ParallelReorderParams {
    int64_t round = 0;     // vertices per dendrogram round (0: max(4096, min(2^20, n / 4096)))
    int64_t segments = 0;  // ordering segments (0: max(1, n / 65536))
    int L = 0;             // candidate window (0: 8)
    ParallelReorderParams();
};
std::vector<uint32_t> reorder_alg1(const Csr &a);

// host/hotcols.cpp -- reading R22: colorig = columns by descending in-degree over the plan's rows
// [r0, r1) of the (reordered) matrix, ties by id.  Without force, applied (returns true) only if
// the 1% most referenced of the referenced columns carry >= kHotSkew of those rows' nnz.
bool hot_column_order(const Csr &a, const std::vector<uint32_t> &perm, int64_t r0, int64_t r1, bool force,
                      std::vector<uint32_t> &colorig);
std::vector<uint32_t> reorder_alg1_parallel(const Csr &a, const ParallelReorderParams &pp);

// kernels (device side, kernels/*.cu)
struct DevicePlan {
    int64_t W = 0, NB = 0, nnz = 0, rows = 0, n_units = 0, n_split = 0, n_segments = 0;
    int precision = 0;
    int wh = kWindow;              // rows per RowWindow (8 = paper; 16/32 tall windows, R20)
    int kernel = ACCSPMM_KERNEL_MMA_SYNC;  // resolved accspmm_kernel
    uint32_t *rwo = nullptr, *tco = nullptr, *a2b = nullptr;
    uint64_t *bits = nullptr;      // [NB][wh/8]
    void *vals = nullptr;
    uint32_t *units = nullptr;     // [n_units][8]
    uint32_t *row_map = nullptr;   // slab row -> C row (nparts == 1 with a permutation), else null
    int hot = 0;                   // 1: hot-column tags in the lane-0 SparseAToB entries (R22)
    uint32_t *orig_map = nullptr;  // slab row -> original row (fused all-gather); = row_map when nparts == 1
    int64_t K = 0;                 // rows of B (padding lanes gather row K -> TMA zero fill)
    // cached TMA tensor maps of the last B operand (key: ptr, N, FW, dtype): one per feature
    // slice (kMaxSliceMaps at most), else one map over all N columns
    mutable uint64_t tmap_key[4] = {0, 0, 0, 0};
    alignas(64) mutable unsigned char tmap[128 * 8] = {};
};

// kernels/build_sm100.cu -- the same BitTCF arrays built by data-parallel device passes
// (SparseAToB padding lanes already hold kPadLane); rwo_host = RowWindowOffset for the
// host-side schedule.  On failure the caller frees what was allocated (free_device_format).
struct DeviceFormat {
    int64_t W = 0, NB = 0, nnz = 0, rows = 0, sum_U = 0;
    int wh = kWindow;
    uint32_t *rwo = nullptr, *tco = nullptr, *a2b = nullptr;
    uint64_t *bits = nullptr;
    void *vals = nullptr;
    std::vector<uint32_t> rwo_host;
    double ms_upload = 0.0, ms_build = 0.0;
};
accspmm_status build_format_device(const Csr &a, const float *vals, const std::vector<uint32_t> &perm,
                                   int64_t row_begin, int64_t row_end, int precision, DeviceFormat &out,
                                   const uint32_t *colmap = nullptr, int wh = kWindow);
void free_device_format(DeviceFormat &f);

// Feature-slice width of one warp for a given N (N % 16 == 0): the widest of 128/64/32/16
// dividing N.  Knobs::fw (variants build, must divide N) overrides it for A/B measurements.
int pick_fw(int64_t N);
// variants build: kernel variants (Knobs::kcfg) that read the 3-byte TF32 image of B (B3)
inline bool is_b3_variant(int kcfg) { return kcfg >= 58 && kcfg <= 61; }

// round_b: the kernel applies rho(B) in registers (B not pre-rounded)
// dst/ndst (ndst > 0): fused all-gather epilogue instead of C (accspmm_execute_allgather)
// b3: B is the 3-byte TF32 image written by launch_pack_b3 (TF32, pre-rounded, slice of 64/128)
accspmm_status launch_spmm(const DevicePlan &p, const void *B, const void *zrow, int64_t N, float *C, float *ws,
                           uint32_t *counters, void *stream, bool round_b, float *const *dst = nullptr,
                           int ndst = 0, bool b3 = false);
// rho(B) -> 3-byte TF32 image (K rows x 3N bytes, per FW slice: FW u16 high halves, FW bytes
// 15..8), rows gathered through perm when non-null (symmetric reordering, R18)
accspmm_status launch_pack_b3(const float *B, void *out, const uint32_t *perm, int64_t K, int64_t N, int FW,
                              void *stream);
// kernels/spmm_tc05_sm100.cu: the tcgen05/TMEM kernel (TF32, N % 128 == 0, any window height)
accspmm_status launch_spmm_tc05(const DevicePlan &d, const void *B, int64_t N, float *C, float *ws, uint32_t *counters,
                                void *stream, bool round_b);
accspmm_status launch_round_b(const float *B, float *Br, int64_t n, void *stream);
#ifdef ACCSPMM_VARIANTS
void debug_tc05_trace(unsigned long long *out);  // [64 CTAs][16]: producer 0-7, transposer 8-15
#endif
// B' = B[perm] row gather (K rows of row_bytes), optionally with rho = TF32 RNA (f32 rows)
accspmm_status launch_permute_b(const void *B, void *Bp, const uint32_t *perm, int64_t K, int64_t row_bytes,
                                bool round_tf32, void *stream);
accspmm_status launch_unpermute(const float *G, const uint32_t *orig_row, int64_t n_rows, int64_t N,
                                float *C, void *stream);
accspmm_status launch_round_tf32(const float *in, float *out, int64_t n, void *stream);
// device SparseAToB (n entries): new column ids -> original ids colorig[], padding kept; levels:
// the hotness tag of each block in its lane-0 entry (kHotShift)
accspmm_status launch_relabel_cols(uint32_t *a2b, int64_t n, const uint32_t *colorig, bool levels, void *stream);
accspmm_status launch_decode(const DevicePlan &p, float *tiles, void *stream);
accspmm_status probe_l2_read(int64_t bytes, int iters, double *gbs, int mode);  // 0 best, 1 LDG, 2 TMA

}  // namespace accspmm
