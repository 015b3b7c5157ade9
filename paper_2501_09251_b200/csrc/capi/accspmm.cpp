// C ABI of libaccspmm (include/accspmm.h): plan lifecycle, device upload, execute.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>

#include "../internal.hpp"

struct accspmm_plan {
    accspmm_plan_info info{};
    accspmm_options opt{};
    accspmm::HostFormat host;           // kept only for host-only plans
    std::vector<uint32_t> units_host;   // [n_units][8]
    std::vector<uint32_t> orig_rows;    // slab row -> original row
    std::vector<uint32_t> colmap;       // relabelled columns (permute_cols, R22): original -> new id
    accspmm::DevicePlan dev{};
    // split-window workspace (grown on demand by execute)
    mutable float *ws = nullptr;
    mutable size_t ws_bytes = 0;
    mutable uint32_t *counters = nullptr;
    mutable size_t counters_n = 0;
    // e2e staging buffers (grown on demand by execute_host / execute_host_batch: two slots)
    mutable void *dB = nullptr;
    mutable size_t dB_bytes = 0;
    mutable float *dC = nullptr;
    mutable size_t dC_bytes = 0;
    mutable void *dB2 = nullptr;      // second slots of the pipelined batch path (own sizes:
    mutable size_t dB2_bytes = 0;     // execute_host grows only the first slots)
    mutable float *dC2 = nullptr;
    mutable size_t dC2_bytes = 0;
    // copy-engine streams and slot events of the pipelined batch path
    mutable cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    mutable cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_k[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    // TF32: rounded copy of B (K x N) produced by the pre-pass of each execute
    mutable float *Br = nullptr;
    mutable size_t Br_bytes = 0;
    // zero row read by padding lanes (>= 128 features x 4 B)
    void *zrow = nullptr;
    // N % 16 != 0: B and C staged through zero-padded K x Np / rows x Np scratch
    mutable void *padB = nullptr;
    mutable size_t padB_bytes = 0;
    mutable float *padC = nullptr;
    mutable size_t padC_bytes = 0;
    // kernel timing ring
    mutable bool timing = false;
    mutable std::vector<cudaEvent_t> ev;
    mutable size_t ev_n = 0;
    mutable std::mutex mu;
};

namespace accspmm {

static thread_local std::string g_last_error;

accspmm_status fail(accspmm_status s, const std::string &msg)
{
    g_last_error = msg;
    return s;
}

static accspmm_status cuda_fail(cudaError_t e, const char *what)
{
    return fail(ACCSPMM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Makes `dev` current for the scope of one entry point and restores the caller's device
// (torch keeps its own notion of the current device; a plan may live on another one).
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev)
    {
        if (dev < 0) return;
        if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; cudaGetLastError(); }
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
        if (!ok) cudaGetLastError();
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;
};

static double ms_since(std::chrono::steady_clock::time_point t0)
{
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// pad = extra zeroed elements after the data (the TMA value window may read up to
// 16 bytes past the last value of a block)
template <class T>
static accspmm_status upload(T **dst, const std::vector<T> &src, int64_t &bytes, size_t pad = 0)
{
    size_t n = (src.size() ? src.size() : 1) + pad;
    cudaError_t e = cudaMalloc((void **)dst, n * sizeof(T));
    if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? fail(ACCSPMM_ERR_OUT_OF_MEMORY, "cudaMalloc")
                                                                : cuda_fail(e, "cudaMalloc");
    bytes += (int64_t)(n * sizeof(T));
    if (pad || src.empty()) cudaMemset(*dst, 0, n * sizeof(T));
    if (!src.empty()) {
        e = cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy H2D");
    }
    return ACCSPMM_OK;
}

static void free_device(accspmm_plan *p)
{
    auto &d = p->dev;
    cudaFree(d.rwo); cudaFree(d.tco); cudaFree(d.a2b); cudaFree(d.bits); cudaFree(d.vals);
    cudaFree(d.units); cudaFree(d.row_map); cudaFree(d.orig_map);
    cudaFree(p->ws); cudaFree(p->counters); cudaFree(p->dB); cudaFree(p->dC); cudaFree(p->Br); cudaFree(p->zrow);
    cudaFree(p->dB2); cudaFree(p->dC2);
    p->dB2 = nullptr; p->dC2 = nullptr;
    p->dB2_bytes = p->dC2_bytes = 0;
    cudaFree(p->padB); cudaFree(p->padC);
    p->padB = nullptr; p->padC = nullptr;
    if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
    if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
    p->s_h2d = p->s_d2h = nullptr;
    for (int k = 0; k < 2; ++k) {
        if (p->ev_in[k]) cudaEventDestroy(p->ev_in[k]);
        if (p->ev_k[k]) cudaEventDestroy(p->ev_k[k]);
        if (p->ev_out[k]) cudaEventDestroy(p->ev_out[k]);
        p->ev_in[k] = p->ev_k[k] = p->ev_out[k] = nullptr;
    }
    for (auto e : p->ev) cudaEventDestroy(e);
    p->ev.clear();
    d = DevicePlan();
    p->ws = nullptr; p->counters = nullptr; p->dB = nullptr; p->dC = nullptr; p->Br = nullptr; p->zrow = nullptr;
    p->ws_bytes = p->counters_n = p->dB_bytes = p->dC_bytes = p->Br_bytes = p->padB_bytes = p->padC_bytes = 0;
}

}  // namespace accspmm

using namespace accspmm;

template <class T>
static accspmm_status export_array(T *dst, const std::vector<T> &host, const T *dev, size_t n)
{
    if (!dst || n == 0) return ACCSPMM_OK;
    if (dev) {
        cudaError_t e = cudaMemcpy(dst, dev, n * sizeof(T), cudaMemcpyDeviceToHost);
        return e == cudaSuccess ? ACCSPMM_OK : cuda_fail(e, "cudaMemcpy D2H");
    }
    std::memcpy(dst, host.data(), n * sizeof(T));
    return ACCSPMM_OK;
}

extern "C" {

accspmm_status accspmm_options_default(accspmm_options *opt)
{
    if (!opt) return fail(ACCSPMM_ERR_INVALID_VALUE, "opt is NULL");
    std::memset(opt, 0, sizeof(*opt));
    opt->precision = ACCSPMM_TF32;
    opt->reorder = ACCSPMM_REORDER_AUTO;  // "defaults: TF32, reorder auto, balance auto"
    opt->balance = ACCSPMM_BALANCE_AUTO;
    opt->unit_cap = 0;
    opt->part = 0;
    opt->nparts = 1;
    int dev = 0;
    opt->device = cudaGetDevice(&dev) == cudaSuccess ? dev : 0;
    cudaGetLastError();
    return ACCSPMM_OK;
}

accspmm_status accspmm_plan_create(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                   const float *vals, accspmm_plan **out)
{
    return accspmm_plan_create_ex(M, K, rowptr, colidx, vals, nullptr, out);
}

static accspmm_status plan_create_impl(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                       const float *vals, const accspmm_options *opt_in, const uint32_t *given_perm,
                                       accspmm_plan **out);

accspmm_status accspmm_plan_create_ex(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                      const float *vals, const accspmm_options *opt_in, accspmm_plan **out)
{
    return plan_create_impl(M, K, rowptr, colidx, vals, opt_in, nullptr, out);
}

accspmm_status accspmm_plan_create_perm(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                        const float *vals, const accspmm_options *opt_in,
                                        const uint32_t *perm_new2old, accspmm_plan **out)
{
    if (!perm_new2old) return fail(ACCSPMM_ERR_INVALID_VALUE, "perm is NULL");
    if (M != K) return fail(ACCSPMM_ERR_INVALID_VALUE, "a row permutation from Alg. 1 needs a square A (Q14)");
    std::vector<char> seen((size_t)M, 0);
    for (int64_t r = 0; r < M; ++r) {
        const uint32_t o = perm_new2old[r];
        if ((int64_t)o >= M || seen[o]) return fail(ACCSPMM_ERR_INVALID_VALUE, "perm is not a bijection of [0, M)");
        seen[o] = 1;
    }
    return plan_create_impl(M, K, rowptr, colidx, vals, opt_in, perm_new2old, out);
}

static accspmm_status plan_create_impl(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                       const float *vals, const accspmm_options *opt_in, const uint32_t *given_perm,
                                       accspmm_plan **out)
{
    if (!out) return fail(ACCSPMM_ERR_INVALID_VALUE, "out is NULL");
    *out = nullptr;
    accspmm_options opt;
    if (opt_in) opt = *opt_in; else accspmm_options_default(&opt);
    if (opt.precision != ACCSPMM_TF32 && opt.precision != ACCSPMM_FP16)
        return fail(ACCSPMM_ERR_INVALID_VALUE, "unknown precision");
    if (opt.reorder < 0 || opt.reorder > 2 || opt.balance < 0 || opt.balance > 2)
        return fail(ACCSPMM_ERR_INVALID_VALUE, "unknown reorder/balance mode");
    if (opt.nparts < 1 || opt.part < 0 || opt.part >= opt.nparts)
        return fail(ACCSPMM_ERR_INVALID_VALUE, "part must be in [0, nparts)");
    if (opt.unit_cap < 0) return fail(ACCSPMM_ERR_INVALID_VALUE, "unit_cap < 0");
    if (opt.build != ACCSPMM_BUILD_HOST && opt.build != ACCSPMM_BUILD_DEVICE)
        return fail(ACCSPMM_ERR_INVALID_VALUE, "unknown build mode");
    if (opt.build == ACCSPMM_BUILD_DEVICE && opt.device < 0)
        return fail(ACCSPMM_ERR_UNSUPPORTED, "device build needs a device (device >= 0)");
    // window height (reading R20): 8 = the paper's BitTCF; 16 / 32 = tall windows (tcgen05 kernel)
    const int wh = opt.window_rows == 0 ? kWindow : opt.window_rows;
    if (wh != 8 && wh != 16 && wh != 32) return fail(ACCSPMM_ERR_INVALID_VALUE, "window_rows must be 0, 8, 16 or 32");
    if (opt.kernel < ACCSPMM_KERNEL_AUTO || opt.kernel > ACCSPMM_KERNEL_TCGEN05)
        return fail(ACCSPMM_ERR_INVALID_VALUE, "unknown kernel");
    if (opt.hot_cols < ACCSPMM_HOT_AUTO || opt.hot_cols > ACCSPMM_HOT_OFF)
        return fail(ACCSPMM_ERR_INVALID_VALUE, "unknown hot_cols mode");
    if (wh > 2 * kWindow && opt.kernel == ACCSPMM_KERNEL_MMA_SYNC)
        return fail(ACCSPMM_ERR_UNSUPPORTED, "the mma.sync kernel runs 8- or 16-row windows");
    // tall windows default to the tcgen05 kernel; kernel = MMA_SYNC runs 16-row windows on the
    // mma.sync kernel (two accumulator halves per gathered row)
    const int kernel = (opt.kernel == ACCSPMM_KERNEL_TCGEN05 || (wh > kWindow && opt.kernel != ACCSPMM_KERNEL_MMA_SYNC))
                           ? ACCSPMM_KERNEL_TCGEN05
                           : ACCSPMM_KERNEL_MMA_SYNC;
    if (kernel == ACCSPMM_KERNEL_TCGEN05 && opt.precision != ACCSPMM_TF32)
        return fail(ACCSPMM_ERR_UNSUPPORTED, "the tcgen05 kernel (and tall windows) is TF32 only");
    if (M < 0 || K < 0) return fail(ACCSPMM_ERR_INVALID_VALUE, "negative matrix dimension");
    if (M >= (int64_t)UINT32_MAX || K >= (int64_t)INT32_MAX)
        return fail(ACCSPMM_ERR_UNSUPPORTED, "M or K too large for 32-bit indices");

    // every device call of plan creation runs on opt.device; the caller's device is restored
    DeviceGuard guard(opt.device);
    if (!guard.ok) return fail(ACCSPMM_ERR_CUDA, "cudaSetDevice(opt.device) failed");
    auto t0 = std::chrono::steady_clock::now();
    Csr a{M, K, rowptr, colidx};
    accspmm_status st = validate_csr(a);
    if (st != ACCSPMM_OK) return st;
    const int64_t nnz = M ? rowptr[M] : 0;
    if (nnz > 0 && !vals) return fail(ACCSPMM_ERR_INVALID_VALUE, "vals is NULL");

    accspmm_plan *p = new (std::nothrow) accspmm_plan();
    if (!p) return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "plan allocation");
    p->opt = opt;
    accspmm_plan_info &I = p->info;
    I.M = M; I.K = K; I.nnz = nnz;
    I.precision = opt.precision; I.part = opt.part; I.nparts = opt.nparts; I.device = opt.device;
    I.ms_validate = ms_since(t0);

    // ---- reordering (Algorithm 1), rows only ----
    t0 = std::chrono::steady_clock::now();
    std::vector<uint32_t> perm;
    I.nb_unreordered = -1;
    if (opt.reorder != ACCSPMM_REORDER_OFF && M == K && M > 0) {
        try {
            // a permutation computed once (e.g. on rank 0 and broadcast) replaces Alg. 1 here
            if (given_perm) perm.assign(given_perm, given_perm + M);
            else perm = reorder_alg1(a);
        } catch (const std::bad_alloc &) {
            delete p;
            return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "reordering");
        }
        if (opt.reorder == ACCSPMM_REORDER_AUTO) {
            int64_t nb0 = count_blocks(a, {}, wh);
            int64_t nb1 = count_blocks(a, perm, wh);
            I.nb_unreordered = nb0;
            if (nb1 >= nb0) perm.clear();
        }
    }
    I.reorder_applied = perm.empty() ? 0 : 1;
    I.ms_reorder = ms_since(t0);

    // ---- partition + BitTCF build ----
    t0 = std::chrono::steady_clock::now();
    int64_t wb0 = 0, wb1 = (M + wh - 1) / wh;
    if (opt.nparts > 1) {
        std::vector<int64_t> b = partition_bounds(a, perm, opt.nparts, wh);
        wb0 = b[(size_t)opt.part];
        wb1 = b[(size_t)opt.part + 1];
    }
    const int64_t r0 = wb0 * wh, r1 = std::min<int64_t>(M, wb1 * wh);
    // Column relabelling: the format is built on A Q^T (colmap = Q^-1: column c -> new id) and the
    // device SparseAToB is mapped back to original ids (colorig = Q), so B is gathered as is.
    //  * symmetric reordering (NEXT-2): Q = the row permutation;
    //  * hot columns (reading R22): Q = columns by descending in-degree over this plan's rows
    //    (ties by id), so every window condenses its hottest columns first.
    std::vector<uint32_t> colmap, colorig;
    if (opt.permute_cols && !perm.empty()) {
        colmap.resize((size_t)M);
        for (int64_t r = 0; r < M; ++r) colmap[perm[(size_t)r]] = (uint32_t)r;
        colorig = perm;
    }
    const bool hot_ok = wh == kWindow && kernel == ACCSPMM_KERNEL_MMA_SYNC && !opt.permute_cols && K > 0 &&
                        K <= (int64_t)kHotIdMask;
    if (opt.hot_cols == ACCSPMM_HOT_ON && !hot_ok) {
        delete p;
        return fail(ACCSPMM_ERR_UNSUPPORTED, "hot_cols: 8-row windows, mma.sync kernel, no permute_cols, K < 2^27");
    }
    if (hot_ok && (opt.hot_cols == ACCSPMM_HOT_ON || (opt.hot_cols == ACCSPMM_HOT_AUTO && K >= kHotMinCols))) {
        if (!hot_column_order(a, perm, r0, std::max(r0, r1), opt.hot_cols == ACCSPMM_HOT_ON, colorig)) colorig.clear();
        if (!colorig.empty()) {
            colmap.resize((size_t)K);
            for (int64_t i = 0; i < K; ++i) colmap[colorig[(size_t)i]] = (uint32_t)i;
        }
    }
    const bool hot = !colorig.empty() && !opt.permute_cols;
    const uint32_t *cm = colmap.empty() ? nullptr : colmap.data();
    I.cols_permuted = (cm && opt.permute_cols) ? 1 : 0;
    I.hot_cols = hot ? 1 : 0;
    HostFormat &F = p->host;
    DeviceFormat DF;
    double ms_csr_upload = 0.0;
    if (opt.build == ACCSPMM_BUILD_DEVICE) {
        st = build_format_device(a, vals, perm, r0, std::max(r0, r1), opt.precision, DF, cm, wh);
        if (st != ACCSPMM_OK) { free_device_format(DF); delete p; return st; }
        F.W = DF.W; F.NB = DF.NB; F.nnz = DF.nnz; F.rows = DF.rows; F.sum_U = DF.sum_U;
        F.rwo = DF.rwo_host;
        ms_csr_upload = DF.ms_upload;
    } else {
        st = build_format(a, vals, perm, r0, std::max(r0, r1), opt.precision, F, cm, wh);
        if (st != ACCSPMM_OK) { delete p; return st; }
    }
    if (I.nb_unreordered < 0 && opt.nparts == 1 && perm.empty()) I.nb_unreordered = F.NB;
    I.rows = F.rows; I.row_begin = r0; I.window_begin = wb0;
    I.W = F.W; I.NB = F.NB; I.plan_nnz = F.nnz; I.sum_U = F.sum_U;
    I.mean_nnz_tc = F.NB ? (double)F.nnz / (double)F.NB : 0.0;
    I.window_rows = wh;
    I.kernel = kernel;
    // P:253 for wh = 8; a tall window's block carries wh/8 occupancy words (2 u32 each)
    I.index_bytes = ((F.rows + wh - 1) / wh + (9 + 2 * (wh / kWindow)) * F.NB + 2) * 4;
    I.metcf_index_bytes = ((F.rows + 7) / 8 + 1 + F.NB + 1 + 8 * F.NB) * 4 + F.nnz;
    I.csr_index_bytes = (F.rows + 1) * 4 + F.nnz * 4;
    I.value_bytes = F.nnz * (opt.precision == ACCSPMM_FP16 ? 2 : 4);
    p->orig_rows.resize((size_t)F.rows);
    for (int64_t r = 0; r < F.rows; ++r)
        p->orig_rows[(size_t)r] = perm.empty() ? (uint32_t)(r0 + r) : perm[(size_t)(r0 + r)];
    I.perm_present = perm.empty() ? 0 : 1;
    I.ms_build = opt.build == ACCSPMM_BUILD_DEVICE ? DF.ms_build : ms_since(t0);

    // ---- IBD + schedule ----
    t0 = std::chrono::steady_clock::now();
    const double ibd = compute_ibd(F.rwo);
    const bool balance = opt.balance == ACCSPMM_BALANCE_ON ||
                         (opt.balance == ACCSPMM_BALANCE_AUTO && ibd > kIbdThreshold);
    const int cap = opt.unit_cap > 0 ? opt.unit_cap : auto_cap(F.NB);
    // reading R7c: grouped (unbalanced) plans concatenate only up to min(cap, 32) blocks under
    // the automatic cap; balanced plans keep the paper's single cap for both rules
    const int gcap = (opt.unit_cap > 0 || balance) ? cap : auto_group_cap(cap);
    // AUTO below the IBD threshold keeps windows whole but groups consecutive ones
    // into a warp's unit (reading R7b); OFF is the paper's one window per unit
    const bool group = !balance && opt.balance == ACCSPMM_BALANCE_AUTO;
    Schedule S = build_schedule(F.rwo, cap, balance, opt.precision, group, gcap, wh);
    I.ibd = ibd; I.balanced = balance ? 1 : 0; I.unit_cap = cap; I.grouped = group ? 1 : 0; I.group_cap = gcap;
    I.n_units = (int64_t)S.units.size(); I.n_split_windows = S.n_split; I.n_segments = S.n_segments;
    p->units_host.resize(S.units.size() * 8);
    std::memcpy(p->units_host.data(), S.units.data(), S.units.size() * sizeof(Unit));
    I.ms_schedule = ms_since(t0);

    // ---- device upload ----
    t0 = std::chrono::steady_clock::now();
    if (opt.device >= 0) {
        DevicePlan &d = p->dev;
        d.W = F.W; d.NB = F.NB; d.nnz = F.nnz; d.rows = F.rows; d.n_units = I.n_units;
        d.n_split = S.n_split; d.n_segments = S.n_segments; d.precision = opt.precision; d.K = K;
        d.wh = wh; d.kernel = kernel;
        int64_t bytes = 0;
        if (opt.build == ACCSPMM_BUILD_DEVICE) {  // format already resident: take ownership
            d.rwo = DF.rwo; d.tco = DF.tco; d.a2b = DF.a2b; d.bits = DF.bits; d.vals = DF.vals;
            DF.rwo = DF.tco = DF.a2b = nullptr; DF.bits = nullptr; DF.vals = nullptr;
            const int64_t es = opt.precision == ACCSPMM_FP16 ? 2 : 4;
            bytes += 4 * (F.W + 1) + 4 * (F.NB + 1) + 32 * std::max<int64_t>(F.NB, 1) +
                     8 * (wh / kWindow) * std::max<int64_t>(F.NB, 1) + es * (F.nnz + 16);
        } else {
            st = upload(&d.rwo, F.rwo, bytes);
            // padding: the tcgen05 kernel bulk-copies 16-byte-aligned supersets of these arrays
            if (st == ACCSPMM_OK) st = upload(&d.tco, F.tco, bytes, 4);
        }
        if (st == ACCSPMM_OK && opt.build != ACCSPMM_BUILD_DEVICE) {
            // device copy: padding lanes (no bit in the block's column-OR) hold 0xFFFFFFFF, an
            // out-of-bounds row the TMA zero-fills; the exported paper format keeps 0
            std::vector<uint32_t> a2b_dev(F.a2b);
            const int nwords = wh / kWindow;
#pragma omp parallel for schedule(static)
            for (int64_t b = 0; b < F.NB; ++b) {
                uint64_t m = 0;
                for (int j = 0; j < nwords; ++j) m |= F.bits[(size_t)b * nwords + j];
                m |= m >> 32;
                m |= m >> 16;
                m |= m >> 8;
                for (int l = 0; l < kWindow; ++l)
                    if (!((m >> l) & 1u)) a2b_dev[(size_t)b * kWindow + (size_t)l] = kPadLane;
            }
            st = upload(&d.a2b, a2b_dev, bytes);
        }
        if (st == ACCSPMM_OK && opt.build != ACCSPMM_BUILD_DEVICE) st = upload(&d.bits, F.bits, bytes, 2);
        if (st == ACCSPMM_OK && opt.build != ACCSPMM_BUILD_DEVICE) {
            if (opt.precision == ACCSPMM_FP16) st = upload((uint16_t **)&d.vals, F.v16, bytes, 16);
            else st = upload((float **)&d.vals, F.v32, bytes, 16);
        }
        if (st == ACCSPMM_OK) st = upload(&d.units, p->units_host, bytes);
        if (st == ACCSPMM_OK && opt.nparts == 1 && !perm.empty()) st = upload(&d.row_map, p->orig_rows, bytes);
        if (st == ACCSPMM_OK && !colorig.empty() && F.NB > 0) {
            // device SparseAToB -> original column ids (+ hotness tags, R22)
            uint32_t *dq = nullptr;
            int64_t qb = 0;
            st = upload(&dq, colorig, qb);
            if (st == ACCSPMM_OK) st = launch_relabel_cols(d.a2b, F.NB * 8, dq, hot, nullptr);
            if (st == ACCSPMM_OK && cudaDeviceSynchronize() != cudaSuccess) st = fail(ACCSPMM_ERR_CUDA, "relabel");
            cudaFree(dq);
        }
        d.hot = hot ? 1 : 0;
        if (st == ACCSPMM_OK && !colorig.empty()) p->colmap = std::move(colmap);  // export: original -> new id
        if (st == ACCSPMM_OK && opt.nparts > 1) st = upload(&d.orig_map, p->orig_rows, bytes);
        if (st == ACCSPMM_OK) {
            std::vector<uint32_t> zeros(256, 0u);  // 1 KB: covers a 128-wide FP32 feature slice
            st = upload((uint32_t **)&p->zrow, zeros, bytes);
        }
        if (st != ACCSPMM_OK) { free_device(p); delete p; return st; }
        I.device_bytes = bytes;
        // the device holds the format now; drop the host copy
        HostFormat empty;
        empty.W = F.W; empty.NB = F.NB; empty.nnz = F.nnz; empty.rows = F.rows; empty.sum_U = F.sum_U; empty.wh = wh;
        F = std::move(empty);
    }
    I.ms_upload = ms_since(t0) + ms_csr_upload;
    *out = p;
    return ACCSPMM_OK;
}

static accspmm_status ensure_workspace(const accspmm_plan *p, int64_t N)
{
    const auto &d = p->dev;
    if (d.n_split == 0) return ACCSPMM_OK;
    size_t need_ws = (size_t)d.n_segments * (size_t)N * (size_t)d.wh * sizeof(float);
    const int64_t fw = d.kernel == ACCSPMM_KERNEL_TCGEN05 ? 128 : pick_fw(N);
    size_t need_cnt = (size_t)d.n_split * (size_t)(N / fw);
    if (need_ws > p->ws_bytes) {
        cudaFree(p->ws);
        p->ws = nullptr;
        p->ws_bytes = 0;
        cudaError_t e = cudaMalloc((void **)&p->ws, need_ws);
        if (e != cudaSuccess) return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "split-window workspace");
        p->ws_bytes = need_ws;
    }
    if (need_cnt > p->counters_n) {
        cudaFree(p->counters);
        p->counters = nullptr;
        p->counters_n = 0;
        cudaError_t e = cudaMalloc((void **)&p->counters, need_cnt * sizeof(uint32_t));
        if (e != cudaSuccess) return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "split-window counters");
        e = cudaMemset(p->counters, 0, need_cnt * sizeof(uint32_t));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemset counters");
        p->counters_n = need_cnt;
    }
    return ACCSPMM_OK;
}

// rho(B) for TF32: one elementwise pass when each B row is gathered many times
// (reuse = sum_w |U_w| / K >= kRoundReuse), else in the kernel's registers.
// Knobs::round_b = 1 (pass) / 2 (kernel) overrides the reuse rule (variants build only).
static bool in_kernel_rounding(const accspmm_plan *p)
{
    const int rmode = knobs().round_b;
    return p->opt.precision == ACCSPMM_TF32 && p->info.K > 0 &&
           (rmode == 2 || (rmode != 1 && p->info.sum_U < kRoundReuse * p->info.K));
}

// Variants build, Knobs::b3 = 1 (measured, not taken: DESIGN.md §7): a pre-rounded TF32 B is
// written as its 3-byte image (bits 31..8 of rho(b); bits 12..0 are zero) and gathered at 3/4
// of the bytes by the mma.sync kernel's 64/128-feature slices.  The product library always
// gathers FP32 rows (Knobs::b3 = 0).
static bool b3_layout(const accspmm_plan *p, int64_t N, int ndst)
{
    return p->opt.precision == ACCSPMM_TF32 && !in_kernel_rounding(p) && p->info.K > 0 &&
           p->dev.kernel != ACCSPMM_KERNEL_TCGEN05 && p->dev.wh == kWindow && knobs().b3 != 0 &&
           (ndst > 0 || knobs().kcfg < 0 || is_b3_variant(knobs().kcfg)) &&
           pick_fw(N) >= 64;
}

static accspmm_status execute_impl(const accspmm_plan *p, const void *B, int64_t N, void *C, float *const *dst,
                                   int ndst, void *stream);

// The feature width the kernels run at: a few wide slices rather than many narrow ones
// (N = 602 or 608 -> 640 = 5 x 128 instead of 19 x 32; measured 72.9 ms at 608 = 19 x 32).
// The tcgen05 kernel runs 128-feature slices (UMMA M = 128) only.
static int64_t padded_width(int64_t N, int kernel)
{
    if (kernel == ACCSPMM_KERNEL_TCGEN05) return (N + 127) / 128 * 128;
    return N <= 16 ? 16 : N <= 32 ? 32 : N <= 64 ? 64 : (N + 127) / 128 * 128;
}

// N % 16 != 0: the kernels take 16-feature multiples, so B is copied into a zero-padded
// K x Np scratch (2-D copy + memset of the pad columns), the product goes to an rows x Np
// scratch and the first N columns are copied into C.  Any N >= 1 and any alignment of B/C.
static accspmm_status execute_padded(const accspmm_plan *p, const void *B, int64_t N, void *C, void *stream)
{
    if (!C || (!B && p->info.K > 0)) return fail(ACCSPMM_ERR_INVALID_VALUE, "B or C is NULL");
    const int64_t Np = padded_width(N, p->dev.kernel);
    const size_t es = p->opt.precision == ACCSPMM_FP16 ? 2 : 4;
    const int64_t out_rows = p->opt.nparts == 1 ? p->info.M : p->info.rows;
    const size_t needB = (size_t)std::max<int64_t>(p->info.K, 1) * (size_t)Np * es;
    const size_t needC = (size_t)std::max<int64_t>(out_rows, 1) * (size_t)Np * sizeof(float);
    {
        std::lock_guard<std::mutex> lk(p->mu);
        if (needB > p->padB_bytes) {
            cudaFree(p->padB); p->padB = nullptr; p->padB_bytes = 0;
            if (cudaMalloc(&p->padB, needB) != cudaSuccess) return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "padded B");
            p->padB_bytes = needB;
        }
        if (needC > p->padC_bytes) {
            cudaFree(p->padC); p->padC = nullptr; p->padC_bytes = 0;
            if (cudaMalloc((void **)&p->padC, needC) != cudaSuccess) return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "padded C");
            p->padC_bytes = needC;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (p->info.K > 0) {
        e = cudaMemset2DAsync((char *)p->padB + N * es, Np * es, 0, (Np - N) * es, p->info.K, s);
        if (e == cudaSuccess) e = cudaMemcpy2DAsync(p->padB, Np * es, B, N * es, N * es, p->info.K, cudaMemcpyDefault, s);
        if (e != cudaSuccess) return cuda_fail(e, "padded B copy");
    }
    accspmm_status st = execute_impl(p, p->padB, Np, p->padC, nullptr, 0, stream);
    if (st != ACCSPMM_OK) return st;
    if (out_rows > 0) {
        e = cudaMemcpy2DAsync(C, N * sizeof(float), p->padC, Np * sizeof(float), N * sizeof(float), out_rows,
                              cudaMemcpyDefault, s);
        if (e != cudaSuccess) return cuda_fail(e, "padded C copy");
    }
    return ACCSPMM_OK;
}

static accspmm_status execute_impl(const accspmm_plan *p, const void *B, int64_t N, void *C, float *const *dst,
                                   int ndst, void *stream)
{
    if (!p) return fail(ACCSPMM_ERR_INVALID_VALUE, "plan is NULL");
    if (p->opt.device < 0) return fail(ACCSPMM_ERR_UNSUPPORTED, "host-only plan cannot execute (no CPU fallback)");
    if (N <= 0) return fail(ACCSPMM_ERR_INVALID_VALUE, "N <= 0");
    if (N % 16 != 0 && ndst > 0) return fail(ACCSPMM_ERR_UNSUPPORTED, "fused all-gather needs N % 16 == 0");
    if (ndst > 0 && p->dev.kernel == ACCSPMM_KERNEL_TCGEN05)
        return fail(ACCSPMM_ERR_UNSUPPORTED, "fused all-gather runs on the mma.sync kernel (8-row windows) only");
    if (padded_width(N, p->dev.kernel) != N && ndst == 0) {
        if (p->info.rows == 0) return ACCSPMM_OK;
        return execute_padded(p, B, N, C, stream);
    }
    if (p->info.rows == 0) return ACCSPMM_OK;
    if (!C || (!B && p->info.K > 0)) return fail(ACCSPMM_ERR_INVALID_VALUE, "B or C is NULL");
    if (((uintptr_t)B & 15) || ((uintptr_t)C & 15)) return fail(ACCSPMM_ERR_INVALID_VALUE, "B and C must be 16-byte aligned");
    std::lock_guard<std::mutex> lk(p->mu);
    accspmm_status st = ensure_workspace(p, N);
    if (st != ACCSPMM_OK) return st;
    const void *Bk = B;
    // rho(B) for TF32: one elementwise pass when each B row is gathered many times
    // (reuse = sum_w |U_w| / K >= 32), else in the kernel's registers.  Relabelled columns
    // (permute_cols, R22) need no pass: the device SparseAToB holds original row ids of B.
    const bool tf32 = p->opt.precision == ACCSPMM_TF32;
    const bool in_kernel_round = in_kernel_rounding(p);
    const bool b3 = b3_layout(p, N, ndst);
    if (tf32 && !in_kernel_round && p->info.K > 0) {
        const size_t need = (size_t)p->info.K * (size_t)N * (b3 ? 3 : 4);
        if (need > p->Br_bytes) {
            cudaFree(p->Br);
            p->Br = nullptr;
            p->Br_bytes = 0;
            if (cudaMalloc((void **)&p->Br, need) != cudaSuccess) return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "B scratch");
            p->Br_bytes = need;
        }
        if (b3)
            st = launch_pack_b3((const float *)B, p->Br, nullptr, p->info.K, N, pick_fw(N), stream);
        else
            st = launch_round_b((const float *)B, p->Br, p->info.K * N, stream);
        if (st != ACCSPMM_OK) return st;
        Bk = p->Br;
    }
    const bool timed = p->timing && p->ev_n + 2 <= p->ev.size();
    // Knobs::l2_persist_mib (variants build only, measurement): mark B as an L2-persisting
    // access-policy window for this launch; the stream attribute and the device's persisting-L2
    // limit are both restored right after the launch
    const int64_t persist_mib = knobs().l2_persist_mib;
    cudaStreamAttrValue prev{};
    bool window = false;
    size_t prev_limit = 0;
    bool limit_changed = false;
    if (persist_mib > 0 && p->info.K > 0) {
        int dev = 0, maxp = 0, maxw = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        const size_t want = std::min<size_t>((size_t)persist_mib << 20, (size_t)maxp);
        if (cudaDeviceGetLimit(&prev_limit, cudaLimitPersistingL2CacheSize) == cudaSuccess && prev_limit != want)
            limit_changed = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess;
        const size_t es = tf32 ? 4 : 2;
        const size_t bytes = std::min<size_t>((size_t)p->info.K * (size_t)N * es, (size_t)maxw);
        cudaStreamGetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &prev);
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.base_ptr = const_cast<void *>(Bk);
        v.accessPolicyWindow.num_bytes = bytes;
        v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)want / (float)std::max<size_t>(bytes, 1));
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        window = cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
        cudaGetLastError();
    }
    if (timed) cudaEventRecord(p->ev[p->ev_n], (cudaStream_t)stream);
    if (p->dev.kernel == ACCSPMM_KERNEL_TCGEN05)
        st = launch_spmm_tc05(p->dev, Bk, N, (float *)C, p->ws, p->counters, stream, in_kernel_round);
    else
        st = launch_spmm(p->dev, Bk, p->zrow, N, (float *)C, p->ws, p->counters, stream, in_kernel_round, dst, ndst, b3);
    if (timed) {
        cudaEventRecord(p->ev[p->ev_n + 1], (cudaStream_t)stream);
        p->ev_n += 2;
    }
    if (window) cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &prev);
    if (limit_changed) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prev_limit);
    return st;
}

accspmm_status accspmm_execute(const accspmm_plan *p, const void *B, int64_t N, void *C, void *stream)
{
    if (!p) return fail(ACCSPMM_ERR_INVALID_VALUE, "plan is NULL");
    DeviceGuard guard(p->opt.device);
    return execute_impl(p, B, N, C, nullptr, 0, stream);
}

accspmm_status accspmm_execute_allgather(const accspmm_plan *p, const void *B, int64_t N, void *const *C_all,
                                         int32_t n_dst, void *stream)
{
    if (n_dst < 1 || n_dst > kMaxGatherDst || !C_all) return fail(ACCSPMM_ERR_INVALID_VALUE, "1 <= n_dst <= 8 required");
    float *dst[kMaxGatherDst] = {};
    for (int32_t k = 0; k < n_dst; ++k) {
        if (!C_all[k] || ((uintptr_t)C_all[k] & 15))
            return fail(ACCSPMM_ERR_INVALID_VALUE, "C_all entries must be non-NULL and 16-byte aligned");
        dst[k] = (float *)C_all[k];
    }
    if (!p) return fail(ACCSPMM_ERR_INVALID_VALUE, "plan is NULL");
    DeviceGuard guard(p->opt.device);
    return execute_impl(p, B, N, dst[0], dst, n_dst, stream);
}

accspmm_status accspmm_execute_host(const accspmm_plan *p, const void *B_host, int64_t N, void *C_host, void *stream)
{
    if (!p) return fail(ACCSPMM_ERR_INVALID_VALUE, "plan is NULL");
    if (p->opt.device < 0) return fail(ACCSPMM_ERR_UNSUPPORTED, "host-only plan cannot execute (no CPU fallback)");
    if (N <= 0) return fail(ACCSPMM_ERR_INVALID_VALUE, "N <= 0");
    if (!C_host || (!B_host && p->info.K > 0)) return fail(ACCSPMM_ERR_INVALID_VALUE, "B or C is NULL");
    const size_t es = p->opt.precision == ACCSPMM_FP16 ? 2 : 4;
    const size_t bB = (size_t)p->info.K * (size_t)N * es;
    const size_t bC = (size_t)p->info.rows * (size_t)N * sizeof(float);
    cudaStream_t s = (cudaStream_t)stream;
    DeviceGuard guard(p->opt.device);
    {
        std::lock_guard<std::mutex> lk(p->mu);
        if (bB > p->dB_bytes) {
            cudaFree(p->dB); p->dB = nullptr; p->dB_bytes = 0;
            if (cudaMalloc(&p->dB, bB) != cudaSuccess) return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "e2e B buffer");
            p->dB_bytes = bB;
        }
        if (bC > p->dC_bytes) {
            cudaFree(p->dC); p->dC = nullptr; p->dC_bytes = 0;
            if (cudaMalloc((void **)&p->dC, bC) != cudaSuccess) return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "e2e C buffer");
            p->dC_bytes = bC;
        }
    }
    cudaError_t e = cudaMemcpyAsync(p->dB, B_host, bB, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "H2D B");
    accspmm_status st = execute_impl(p, p->dB, N, p->dC, nullptr, 0, stream);
    if (st != ACCSPMM_OK) return st;
    e = cudaMemcpyAsync(C_host, p->dC, bC, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "D2H C");
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    return ACCSPMM_OK;
}

accspmm_status accspmm_execute_host_batch(const accspmm_plan *p, const void *const *B_hosts, void *const *C_hosts,
                                          int32_t count, int64_t N, void *stream)
{
    if (!p) return fail(ACCSPMM_ERR_INVALID_VALUE, "plan is NULL");
    if (p->opt.device < 0) return fail(ACCSPMM_ERR_UNSUPPORTED, "host-only plan cannot execute (no CPU fallback)");
    if (N <= 0) return fail(ACCSPMM_ERR_INVALID_VALUE, "N <= 0");
    if (count < 0 || (count > 0 && (!B_hosts || !C_hosts))) return fail(ACCSPMM_ERR_INVALID_VALUE, "bad batch");
    for (int32_t i = 0; i < count; ++i)
        if (!C_hosts[i] || (!B_hosts[i] && p->info.K > 0)) return fail(ACCSPMM_ERR_INVALID_VALUE, "B or C is NULL");
    if (count == 0) return ACCSPMM_OK;
    const size_t es = p->opt.precision == ACCSPMM_FP16 ? 2 : 4;
    const size_t bB = (size_t)p->info.K * (size_t)N * es;
    const size_t bC = (size_t)p->info.rows * (size_t)N * sizeof(float);
    cudaStream_t s = (cudaStream_t)stream;
    DeviceGuard guard(p->opt.device);
    {
        std::lock_guard<std::mutex> lk(p->mu);
        // every slot carries its own size (execute_host grows only the first slots)
        auto grow = [&](void **a, size_t &have, size_t need) -> bool {
            if (need <= have && *a) return true;
            cudaFree(*a);
            *a = nullptr;
            have = 0;
            if (cudaMalloc(a, need ? need : 16) != cudaSuccess) {
                *a = nullptr;
                return false;
            }
            have = need;
            return true;
        };
        if (!grow(&p->dB, p->dB_bytes, bB) || !grow(&p->dB2, p->dB2_bytes, bB))
            return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "e2e B buffers");
        if (!grow((void **)&p->dC, p->dC_bytes, bC) || !grow((void **)&p->dC2, p->dC2_bytes, bC))
            return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "e2e C buffers");
        if (!p->s_h2d) {
            cudaError_t e = cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking);
            for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
                e = cudaEventCreateWithFlags(&p->ev_in[k], cudaEventDisableTiming);
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_k[k], cudaEventDisableTiming);
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_out[k], cudaEventDisableTiming);
            }
            if (e != cudaSuccess) return cuda_fail(e, "batch streams/events");
        }
    }
    void *dB[2] = {p->dB, p->dB2};
    float *dC[2] = {p->dC, p->dC2};
    // start after the caller's prior work on `stream`
    cudaError_t e = cudaEventRecord(p->ev_k[0], s);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev_k[1], s);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev_out[0], s);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev_out[1], s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    // three-stage pipeline over two slots: H2D(i+1) and D2H(i-1) overlap the SpMM of step i
    for (int32_t i = 0; i < count; ++i) {
        const int k = i & 1;
        e = cudaStreamWaitEvent(p->s_h2d, p->ev_k[k], 0);  // the SpMM of step i-2 has read dB[k]
        if (e == cudaSuccess) e = cudaMemcpyAsync(dB[k], B_hosts[i], bB, cudaMemcpyHostToDevice, p->s_h2d);
        if (e == cudaSuccess) e = cudaEventRecord(p->ev_in[k], p->s_h2d);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, p->ev_in[k], 0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, p->ev_out[k], 0);  // D2H of step i-2 has read dC[k]
        if (e != cudaSuccess) return cuda_fail(e, "batch H2D");
        accspmm_status st = execute_impl(p, dB[k], N, dC[k], nullptr, 0, stream);
        if (st != ACCSPMM_OK) return st;
        e = cudaEventRecord(p->ev_k[k], s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_d2h, p->ev_k[k], 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(C_hosts[i], dC[k], bC, cudaMemcpyDeviceToHost, p->s_d2h);
        if (e == cudaSuccess) e = cudaEventRecord(p->ev_out[k], p->s_d2h);
        if (e != cudaSuccess) return cuda_fail(e, "batch D2H");
    }
    e = cudaStreamSynchronize(p->s_d2h);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    return ACCSPMM_OK;
}

void accspmm_plan_destroy(accspmm_plan *p)
{
    if (!p) return;
    if (p->opt.device >= 0) {
        DeviceGuard guard(p->opt.device);
        free_device(p);
    }
    delete p;
}

accspmm_status accspmm_plan_get_info(const accspmm_plan *p, accspmm_plan_info *info)
{
    if (!p || !info) return fail(ACCSPMM_ERR_INVALID_VALUE, "NULL argument");
    *info = p->info;
    return ACCSPMM_OK;
}

accspmm_status accspmm_plan_b_bytes(const accspmm_plan *p, int64_t N, int32_t *bytes_per_element)
{
    if (!p || !bytes_per_element) return fail(ACCSPMM_ERR_INVALID_VALUE, "NULL argument");
    if (N <= 0) return fail(ACCSPMM_ERR_INVALID_VALUE, "N <= 0");
    // widths outside 16/32/64/128k run through the padded copy at the next efficient width
    const int64_t Np = padded_width(N, p->dev.kernel);
    *bytes_per_element = p->opt.precision == ACCSPMM_FP16 ? 2 : (b3_layout(p, Np, 0) ? 3 : 4);
    return ACCSPMM_OK;
}

accspmm_status accspmm_plan_export_format(const accspmm_plan *p, uint32_t *rwo, uint32_t *tco, uint32_t *a2b,
                                          uint64_t *bits, void *vals)
{
    if (!p) return fail(ACCSPMM_ERR_INVALID_VALUE, "plan is NULL");
    const auto &I = p->info;
    const bool dev = p->opt.device >= 0;
    DeviceGuard guard(p->opt.device);
    accspmm_status st = export_array(rwo, p->host.rwo, dev ? p->dev.rwo : nullptr, (size_t)I.W + 1);
    if (st == ACCSPMM_OK) st = export_array(tco, p->host.tco, dev ? p->dev.tco : nullptr, (size_t)I.NB + 1);
    if (st == ACCSPMM_OK) {
        st = export_array(a2b, p->host.a2b, dev ? p->dev.a2b : nullptr, (size_t)I.NB * 8);
        // device copy -> the paper format: padding marker -> 0; relabelled columns
        // (permute_cols, R22) hold original ids (+ hotness tags on lane 0) -> the format's new ids
        if (st == ACCSPMM_OK && a2b && dev)
            for (size_t q = 0; q < (size_t)I.NB * 8; ++q) {
                uint32_t v = a2b[q];
                if (v == kPadLane) { a2b[q] = 0u; continue; }
                if (p->dev.hot && (q & 7) == 0) v &= kHotIdMask;
                a2b[q] = p->colmap.empty() ? v : p->colmap[v];
            }
    }
    if (st == ACCSPMM_OK)
        st = export_array(bits, p->host.bits, dev ? p->dev.bits : nullptr, (size_t)I.NB * (size_t)(I.window_rows / kWindow));
    if (st == ACCSPMM_OK) {
        if (p->opt.precision == ACCSPMM_FP16)
            st = export_array((uint16_t *)vals, p->host.v16, dev ? (const uint16_t *)p->dev.vals : nullptr,
                              (size_t)I.plan_nnz);
        else
            st = export_array((float *)vals, p->host.v32, dev ? (const float *)p->dev.vals : nullptr,
                              (size_t)I.plan_nnz);
    }
    return st;
}

accspmm_status accspmm_plan_export_units(const accspmm_plan *p, uint32_t *units)
{
    if (!p || !units) return fail(ACCSPMM_ERR_INVALID_VALUE, "NULL argument");
    std::memcpy(units, p->units_host.data(), p->units_host.size() * sizeof(uint32_t));
    return ACCSPMM_OK;
}

accspmm_status accspmm_plan_export_rows(const accspmm_plan *p, uint32_t *orig_row)
{
    if (!p || !orig_row) return fail(ACCSPMM_ERR_INVALID_VALUE, "NULL argument");
    std::memcpy(orig_row, p->orig_rows.data(), p->orig_rows.size() * sizeof(uint32_t));
    return ACCSPMM_OK;
}

accspmm_status accspmm_reorder(int64_t n, const int64_t *rowptr, const int32_t *colidx, uint32_t *perm_new2old)
{
    if (n < 0 || !perm_new2old) return fail(ACCSPMM_ERR_INVALID_VALUE, "bad argument");
    Csr a{n, n, rowptr, colidx};
    accspmm_status st = validate_csr(a);
    if (st != ACCSPMM_OK) return st;
    try {
        std::vector<uint32_t> perm = reorder_alg1(a);
        std::memcpy(perm_new2old, perm.data(), perm.size() * sizeof(uint32_t));
    } catch (const std::bad_alloc &) {
        return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "reordering");
    }
    return ACCSPMM_OK;
}

accspmm_status accspmm_reorder_parallel(int64_t n, const int64_t *rowptr, const int32_t *colidx, int64_t round,
                                        int64_t segments, int32_t L, uint32_t *perm_new2old)
{
    if (n < 0 || !perm_new2old) return fail(ACCSPMM_ERR_INVALID_VALUE, "bad argument");
    Csr a{n, n, rowptr, colidx};
    accspmm_status st = validate_csr(a);
    if (st != ACCSPMM_OK) return st;
    try {
        ParallelReorderParams pp;
        pp.round = round;
        pp.segments = segments;
        pp.L = L;
        std::vector<uint32_t> perm = reorder_alg1_parallel(a, pp);
        std::memcpy(perm_new2old, perm.data(), perm.size() * sizeof(uint32_t));
    } catch (const std::bad_alloc &) {
        return fail(ACCSPMM_ERR_OUT_OF_MEMORY, "reordering");
    }
    return ACCSPMM_OK;
}

accspmm_status accspmm_csr_transpose(int64_t M, int64_t K, const int64_t *rowptr, const int32_t *colidx,
                                    const float *vals, int64_t *t_rowptr, int32_t *t_colidx, float *t_vals)
{
    if (M < 0 || K < 0 || !t_rowptr) return fail(ACCSPMM_ERR_INVALID_VALUE, "bad argument");
    if (K >= (int64_t)INT32_MAX || M >= (int64_t)INT32_MAX) return fail(ACCSPMM_ERR_UNSUPPORTED, "too large");
    Csr a{M, K, rowptr, colidx};
    accspmm_status st = validate_csr(a);
    if (st != ACCSPMM_OK) return st;
    const int64_t nnz = M ? rowptr[M] : 0;
    if (nnz > 0 && !t_colidx) return fail(ACCSPMM_ERR_INVALID_VALUE, "t_colidx is NULL");
    csr_transpose(a, vals, t_rowptr, t_colidx, t_vals);
    return ACCSPMM_OK;
}

accspmm_status accspmm_partition_bounds(int64_t M, const int64_t *rowptr, int32_t nparts, int64_t *bounds)
{
    if (M < 0 || nparts < 1 || !bounds || (M > 0 && !rowptr)) return fail(ACCSPMM_ERR_INVALID_VALUE, "bad argument");
    Csr a{M, 0, rowptr, nullptr};
    std::vector<int64_t> b = partition_bounds(a, {}, nparts);
    std::memcpy(bounds, b.data(), b.size() * sizeof(int64_t));
    return ACCSPMM_OK;
}

accspmm_status accspmm_plan_set_timing(accspmm_plan *p, int32_t enable)
{
    if (!p) return fail(ACCSPMM_ERR_INVALID_VALUE, "plan is NULL");
    if (p->opt.device < 0) return fail(ACCSPMM_ERR_UNSUPPORTED, "host-only plan");
    DeviceGuard guard(p->opt.device);
    std::lock_guard<std::mutex> lk(p->mu);
    if (enable && p->ev.empty()) {
        p->ev.resize(8192);
        for (auto &e : p->ev)
            if (cudaEventCreate(&e) != cudaSuccess) return cuda_fail(cudaGetLastError(), "cudaEventCreate");
    }
    p->timing = enable != 0;
    p->ev_n = 0;
    return ACCSPMM_OK;
}

accspmm_status accspmm_plan_kernel_times(accspmm_plan *p, float *ms_out, int32_t max_n, int32_t *n_out)
{
    if (!p || !n_out || (max_n > 0 && !ms_out)) return fail(ACCSPMM_ERR_INVALID_VALUE, "NULL argument");
    std::lock_guard<std::mutex> lk(p->mu);
    int32_t n = 0;
    for (size_t k = 0; k + 1 < p->ev_n && n < max_n; k += 2) {
        cudaError_t e = cudaEventSynchronize(p->ev[k + 1]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
        float ms = 0.f;
        e = cudaEventElapsedTime(&ms, p->ev[k], p->ev[k + 1]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
        ms_out[n++] = ms;
    }
    p->ev_n = 0;
    *n_out = n;
    return ACCSPMM_OK;
}

accspmm_status accspmm_unpermute(const float *G, const uint32_t *orig_row, int64_t n_rows, int64_t N, float *C,
                                 void *stream)
{
    if (n_rows < 0 || N <= 0 || N % 4 != 0) return fail(ACCSPMM_ERR_INVALID_VALUE, "bad size");
    if (n_rows == 0) return ACCSPMM_OK;
    if (!G || !orig_row || !C) return fail(ACCSPMM_ERR_INVALID_VALUE, "NULL pointer");
    return launch_unpermute(G, orig_row, n_rows, N, C, stream);
}

accspmm_status accspmm_debug_round_tf32(const float *in, float *out, int64_t n, void *stream)
{
    if (n < 0 || (n > 0 && (!in || !out))) return fail(ACCSPMM_ERR_INVALID_VALUE, "bad argument");
    if (n == 0) return ACCSPMM_OK;
    return launch_round_tf32(in, out, n, stream);
}

accspmm_status accspmm_debug_decode(const accspmm_plan *p, float *tiles, void *stream)
{
    if (!p) return fail(ACCSPMM_ERR_INVALID_VALUE, "plan is NULL");
    if (p->opt.device < 0) return fail(ACCSPMM_ERR_UNSUPPORTED, "host-only plan");
    if (p->info.NB == 0) return ACCSPMM_OK;
    if (!tiles) return fail(ACCSPMM_ERR_INVALID_VALUE, "tiles is NULL");
    DeviceGuard guard(p->opt.device);
    return launch_decode(p->dev, tiles, stream);
}

accspmm_status accspmm_probe_l2_bandwidth(int64_t bytes, int32_t iters, double *gbs)
{
    if (bytes < (1 << 20) || iters < 1 || !gbs) return fail(ACCSPMM_ERR_INVALID_VALUE, "bad argument");
    return probe_l2_read(bytes & ~(int64_t)15, iters, gbs, 1);
}

accspmm_status accspmm_probe_l2_bandwidth_ex(int64_t bytes, int32_t iters, int32_t mode, double *gbs)
{
    if (bytes < (1 << 20) || iters < 1 || !gbs || mode < 0 || mode > 2)
        return fail(ACCSPMM_ERR_INVALID_VALUE, "bad argument");
    return probe_l2_read(bytes & ~(int64_t)16383, iters, gbs, mode);
}

const char *accspmm_status_string(accspmm_status s)
{
    switch (s) {
    case ACCSPMM_OK: return "ACCSPMM_OK";
    case ACCSPMM_ERR_INVALID_VALUE: return "ACCSPMM_ERR_INVALID_VALUE";
    case ACCSPMM_ERR_INVALID_CSR: return "ACCSPMM_ERR_INVALID_CSR";
    case ACCSPMM_ERR_UNSUPPORTED: return "ACCSPMM_ERR_UNSUPPORTED";
    case ACCSPMM_ERR_OUT_OF_MEMORY: return "ACCSPMM_ERR_OUT_OF_MEMORY";
    case ACCSPMM_ERR_CUDA: return "ACCSPMM_ERR_CUDA";
    case ACCSPMM_ERR_INTERNAL: return "ACCSPMM_ERR_INTERNAL";
    }
    return "ACCSPMM_UNKNOWN_STATUS";
}

const char *accspmm_last_error(void) { return g_last_error.c_str(); }

int32_t accspmm_abi_version(void) { return ACCSPMM_ABI_VERSION; }

#ifdef ACCSPMM_VARIANTS
// measurement hook of the variants build: per-phase cycle trace of the tcgen05 kernel (kcfg 68)
void accspmm_debug_tc05_trace(unsigned long long *out) { accspmm::debug_tc05_trace(out); }
#endif

}  // extern "C"
