// Device-side BitTCF builder (plan option build = ACCSPMM_BUILD_DEVICE).
//
// Builds the same five arrays as the host builder (host/bittcf.cpp, §3.3,
// P:248-273) straight into device memory, as a sequence of data-parallel passes
// instead of a per-window loop:
//
//   1. slab row lengths through the row permutation, exclusive scan -> slab CSR offsets
//   2. one 64-bit key per nnz: (window, column, row-in-window); rho(value) as payload
//   3. radix sort of the keys (cub) -- a window's entries stay in its CSR range, now
//      ordered by column: the window's condensed columns are the column runs
//   4. run heads + inclusive scan -> per-nnz condensed position inside its window
//   5. per window |U_w| -> ceil(|U_w|/8) blocks, exclusive scan -> RowWindowOffset
//   6. per nnz: SparseAToB[8b + lane] = column at run heads, TCLocalBit bit
//      r*8 + lane set with atomicOr (reading Q3)
//   7. popcount per block, exclusive scan -> TCOffset
//   8. per nnz: value index = TCOffset[b] + popc(mask & (2^k - 1)) (P:273 in reverse)
//
// Padding lanes of SparseAToB get the device marker kPadLane directly (reading R17).
// Tall windows (wh = 16 / 32 rows, reading R20): the row-in-window field of the key has
// log2(wh) bits, a block owns wh/8 occupancy words (word = row / 8, bit = (row % 8) * 8 + lane)
// and a value's index adds the popcounts of the block's earlier words.
// Every array is a pure function of the input, so the device build equals the host build
// bit for bit (tests/test_gpu_build.py).
#include <cub/cub.cuh>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>

#include "../internal.hpp"

namespace accspmm {
namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(int64_t n, int per_thread = 1)
{
    int64_t g = (n + (int64_t)kThreads * per_thread - 1) / ((int64_t)kThreads * per_thread);
    if (g > 148 * 64) g = 148 * 64;
    return (unsigned)(g < 1 ? 1 : g);
}

inline int bits_for(uint64_t maxval)  // bits needed to hold values 0..maxval
{
    int b = 0;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}

// rho on the device, matching host/csr.cpp bit for bit: TF32 = cvt.rna.tf32.f32 (NaN
// payloads truncated, reading R1); FP16 = round-to-nearest-even, NaN -> quiet NaN with the
// top payload bits (the host compiler's conversion)
__device__ __forceinline__ uint32_t rho_bits(float x, bool f16)
{
    if (!f16) {
        uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
        return r;
    }
    const uint32_t u = __float_as_uint(x);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu) != 0u)
        return ((u >> 16) & 0x8000u) | 0x7E00u | ((u >> 13) & 0x3FFu);
    return (uint32_t)__half_as_ushort(__float2half_rn(x));
}

__global__ void row_len_kernel(const int64_t *__restrict__ rowptr, const uint32_t *__restrict__ perm, int64_t r0,
                               int64_t rows, int64_t *__restrict__ len)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = perm ? (int64_t)perm[r0 + r] : r0 + r;
        len[r] = rowptr[o + 1] - rowptr[o];
    }
}

// one warp per slab row: key = window << (cbits + lw) | col << lw | row-in-window (wh = 2^lw)
__global__ void keys_kernel(const int64_t *__restrict__ rowptr, const int32_t *__restrict__ colidx,
                            const float *__restrict__ vals, const uint32_t *__restrict__ perm, int64_t r0, int64_t rows,
                            const int64_t *__restrict__ sptr, int cbits, int lw, bool f16,
                            const uint32_t *__restrict__ colmap, uint64_t *__restrict__ keys, uint32_t *__restrict__ vbits)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
        const int64_t o = perm ? (int64_t)perm[r0 + r] : r0 + r;
        const int64_t p0 = rowptr[o], n = rowptr[o + 1] - p0, q0 = sptr[r];
        const uint64_t hi = ((uint64_t)(r >> lw) << (cbits + lw)) | (uint64_t)(r & ((1 << lw) - 1));
        for (int64_t i = lane; i < n; i += 32) {
            const uint32_t c = (uint32_t)colidx[p0 + i];
            keys[q0 + i] = hi | ((uint64_t)(colmap ? colmap[c] : c) << lw);
            vbits[q0 + i] = rho_bits(vals[p0 + i], f16);
        }
    }
}

// run heads of the sorted keys (a new (window, column) pair)
struct HeadOp {
    const uint64_t *keys;
    int lw;
    __host__ __device__ __forceinline__ uint32_t operator()(int64_t i) const
    {
        return (i == 0 || (keys[i] >> lw) != (keys[i - 1] >> lw)) ? 1u : 0u;
    }
};

// per window: ustart (unique columns before it) and blocks = ceil(|U_w| / 8)
__global__ void window_kernel(const int64_t *__restrict__ sptr, const uint32_t *__restrict__ uid, int64_t W,
                              int64_t rows, int wh, uint32_t *__restrict__ ustart, uint32_t *__restrict__ blocks)
{
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < W; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = sptr[w * wh], hi = sptr[min(rows, w * wh + wh)];
        const uint32_t us = lo > 0 ? uid[lo - 1] : 0u;
        const uint32_t U = hi > lo ? uid[hi - 1] - us : 0u;
        ustart[w] = us;
        blocks[w] = (U + 7u) >> 3;
    }
}

// block b, occupancy word, bit inside the word, column and lane of one sorted key
__device__ __forceinline__ void locate(uint64_t key, uint32_t u, int cbits, int lw, const uint32_t *ustart,
                                       const uint32_t *rwo, uint32_t &b, int &word, int &k, uint32_t &col,
                                       uint32_t &lane)
{
    const uint64_t w = key >> (cbits + lw);
    col = (uint32_t)((key >> lw) & ((1ull << cbits) - 1ull));
    const uint32_t pos = u - 1u - ustart[w];
    const int rloc = (int)(key & ((1ull << lw) - 1ull));
    lane = pos & 7u;
    b = rwo[w] + (pos >> 3);
    word = rloc >> 3;
    k = (rloc & 7) * 8 + (int)lane;
}

__global__ void fill_kernel(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ uid, int64_t nnz, int cbits,
                            int lw, const uint32_t *__restrict__ ustart, const uint32_t *__restrict__ rwo,
                            uint32_t *__restrict__ a2b, unsigned long long *__restrict__ bits)
{
    const int nw = 1 << (lw - 3);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[i];
        const uint32_t u = uid[i];
        uint32_t b, col, lane;
        int word, k;
        locate(key, u, cbits, lw, ustart, rwo, b, word, k, col, lane);
        if (i == 0 || (keys[i - 1] >> lw) != (key >> lw)) a2b[(size_t)b * 8 + lane] = col;
        atomicOr(bits + (size_t)b * nw + word, 1ull << k);
    }
}

__global__ void popc_kernel(const unsigned long long *__restrict__ bits, int64_t NB, int nw, uint32_t *__restrict__ cnt)
{
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < NB; b += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c = 0;
        for (int j = 0; j < nw; ++j) c += (uint32_t)__popcll(bits[b * nw + j]);
        cnt[b] = c;
    }
}

__global__ void values_kernel(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ uid,
                              const uint32_t *__restrict__ vb, int64_t nnz, int cbits, int lw,
                              const uint32_t *__restrict__ ustart, const uint32_t *__restrict__ rwo,
                              const unsigned long long *__restrict__ bits, const uint32_t *__restrict__ tco, bool f16,
                              void *__restrict__ vals)
{
    const int nw = 1 << (lw - 3);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t b, col, lane;
        int word, k;
        locate(keys[i], uid[i], cbits, lw, ustart, rwo, b, word, k, col, lane);
        uint32_t idx = tco[b] + (uint32_t)__popcll(bits[(size_t)b * nw + word] & ((1ull << k) - 1ull));
        for (int j = 0; j < word; ++j) idx += (uint32_t)__popcll(bits[(size_t)b * nw + j]);
        if (f16) reinterpret_cast<uint16_t *>(vals)[idx] = (uint16_t)vb[i];
        else reinterpret_cast<uint32_t *>(vals)[idx] = vb[i];
    }
}

// RAII scratch allocation (freed on every exit path)
struct Scratch {
    void *p = nullptr;
    ~Scratch() { cudaFree(p); }
    template <class T>
    T *get() const { return reinterpret_cast<T *>(p); }
};

struct Builder {
    cudaStream_t s = nullptr;
    accspmm_status st = ACCSPMM_OK;
    bool ok(cudaError_t e, const char *what)
    {
        if (e == cudaSuccess) return true;
        st = fail(e == cudaErrorMemoryAllocation ? ACCSPMM_ERR_OUT_OF_MEMORY : ACCSPMM_ERR_CUDA,
                  std::string("device build: ") + what + ": " + cudaGetErrorString(e));
        cudaGetLastError();
        return false;
    }
    bool alloc(Scratch &x, size_t bytes, const char *what) { return ok(cudaMalloc(&x.p, bytes ? bytes : 16), what); }
};

}  // namespace

accspmm_status build_format_device(const Csr &a, const float *vals, const std::vector<uint32_t> &perm, int64_t row_begin,
                                   int64_t row_end, int precision, DeviceFormat &out, const uint32_t *colmap, int wh)
{
    using clk = std::chrono::steady_clock;
    const auto t_start = clk::now();
    const int64_t rows = row_end - row_begin;
    const int64_t W = (rows + wh - 1) / wh;
    const int lw = wh == 32 ? 5 : wh == 16 ? 4 : 3;
    const int nwords = wh / kWindow;
    const int64_t nnz_all = a.M ? a.rowptr[a.M] : 0;
    const bool f16 = precision == ACCSPMM_FP16;
    out = DeviceFormat();
    out.rows = rows;
    out.W = W;
    out.wh = wh;
    Builder B;
    if (!B.ok(cudaStreamCreateWithFlags(&B.s, cudaStreamNonBlocking), "stream")) return B.st;
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{B.s};

    // ---- upload the CSR (whole matrix: a slab's rows are scattered by the permutation)
    Scratch d_rowptr, d_colidx, d_vals, d_perm;
    if (!B.alloc(d_rowptr, (size_t)(a.M + 1) * 8, "rowptr") || !B.alloc(d_colidx, (size_t)nnz_all * 4, "colidx") ||
        !B.alloc(d_vals, (size_t)nnz_all * 4, "vals"))
        return B.st;
    if (!B.ok(cudaMemcpyAsync(d_rowptr.p, a.rowptr, (size_t)(a.M + 1) * 8, cudaMemcpyHostToDevice, B.s), "H2D") ||
        (nnz_all && !B.ok(cudaMemcpyAsync(d_colidx.p, a.colidx, (size_t)nnz_all * 4, cudaMemcpyHostToDevice, B.s), "H2D")) ||
        (nnz_all && !B.ok(cudaMemcpyAsync(d_vals.p, vals, (size_t)nnz_all * 4, cudaMemcpyHostToDevice, B.s), "H2D")))
        return B.st;
    if (!perm.empty()) {
        if (!B.alloc(d_perm, perm.size() * 4, "perm") ||
            !B.ok(cudaMemcpyAsync(d_perm.p, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice, B.s), "H2D"))
            return B.st;
    }
    Scratch d_colmap;
    if (colmap) {
        if (!B.alloc(d_colmap, (size_t)a.K * 4, "colmap") ||
            !B.ok(cudaMemcpyAsync(d_colmap.p, colmap, (size_t)a.K * 4, cudaMemcpyHostToDevice, B.s), "H2D"))
            return B.st;
    }
    if (!B.ok(cudaStreamSynchronize(B.s), "upload")) return B.st;
    out.ms_upload = std::chrono::duration<double, std::milli>(clk::now() - t_start).count();
    const auto t_build = clk::now();

    // ---- 1. slab CSR offsets
    Scratch d_len, d_sptr, d_tmp;
    if (!B.alloc(d_len, (size_t)(rows + 1) * 8, "len") || !B.alloc(d_sptr, (size_t)(rows + 1) * 8, "sptr")) return B.st;
    const uint32_t *permp = perm.empty() ? nullptr : d_perm.get<uint32_t>();
    if (rows > 0)
        row_len_kernel<<<grid_for(rows), kThreads, 0, B.s>>>(d_rowptr.get<int64_t>(), permp, row_begin, rows,
                                                             d_len.get<int64_t>());
    if (!B.ok(cudaMemsetAsync(d_len.get<int64_t>() + rows, 0, 8, B.s), "memset")) return B.st;
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_len.get<int64_t>(), d_sptr.get<int64_t>(), rows + 1, B.s);
    if (!B.alloc(d_tmp, tmp_bytes, "scan tmp")) return B.st;
    if (!B.ok(cub::DeviceScan::ExclusiveSum(d_tmp.p, tmp_bytes, d_len.get<int64_t>(), d_sptr.get<int64_t>(), rows + 1,
                                            B.s), "scan"))
        return B.st;
    int64_t nnz = 0;
    if (!B.ok(cudaMemcpyAsync(&nnz, d_sptr.get<int64_t>() + rows, 8, cudaMemcpyDeviceToHost, B.s), "D2H") ||
        !B.ok(cudaStreamSynchronize(B.s), "sync"))
        return B.st;
    if (nnz >= (int64_t)UINT32_MAX) return fail(ACCSPMM_ERR_UNSUPPORTED, "plan nnz overflows u32 TCOffset");
    out.nnz = nnz;

    // ---- 2-3. keys, sort
    const int cbits = a.K > 1 ? bits_for((uint64_t)(a.K - 1)) : 1;
    const int wbits = W > 1 ? bits_for((uint64_t)(W - 1)) : 1;
    if (cbits + wbits + lw > 64) return fail(ACCSPMM_ERR_UNSUPPORTED, "window/column key does not fit 64 bits");
    Scratch d_k0, d_k1, d_v0, d_v1, d_uid, d_sort_tmp;
    if (!B.alloc(d_k0, (size_t)nnz * 8, "keys") || !B.alloc(d_k1, (size_t)nnz * 8, "keys") ||
        !B.alloc(d_v0, (size_t)nnz * 4, "vbits") || !B.alloc(d_v1, (size_t)nnz * 4, "vbits"))
        return B.st;
    if (rows > 0 && nnz > 0)
        keys_kernel<<<grid_for(rows * 32), kThreads, 0, B.s>>>(d_rowptr.get<int64_t>(), d_colidx.get<int32_t>(),
                                                               d_vals.get<float>(), permp, row_begin, rows,
                                                               d_sptr.get<int64_t>(), cbits, lw, f16,
                                                               colmap ? d_colmap.get<uint32_t>() : nullptr,
                                                               d_k0.get<uint64_t>(), d_v0.get<uint32_t>());
    cub::DoubleBuffer<uint64_t> kb(d_k0.get<uint64_t>(), d_k1.get<uint64_t>());
    cub::DoubleBuffer<uint32_t> vb(d_v0.get<uint32_t>(), d_v1.get<uint32_t>());
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, kb, vb, nnz, 0, cbits + wbits + lw, B.s);
    if (!B.alloc(d_sort_tmp, sort_bytes, "sort tmp")) return B.st;
    if (nnz > 0 && !B.ok(cub::DeviceRadixSort::SortPairs(d_sort_tmp.p, sort_bytes, kb, vb, nnz, 0, cbits + wbits + lw, B.s),
                         "radix sort"))
        return B.st;
    const uint64_t *keys = kb.Current();
    const uint32_t *vbits = vb.Current();

    // ---- 4. run heads -> uid (1-based rank of the (window, column) run)
    if (!B.alloc(d_uid, (size_t)nnz * 4, "uid")) return B.st;
    cub::TransformInputIterator<uint32_t, HeadOp, cub::CountingInputIterator<int64_t>> heads(
        cub::CountingInputIterator<int64_t>(0), HeadOp{keys, lw});
    size_t scan2 = 0;
    cub::DeviceScan::InclusiveSum(nullptr, scan2, heads, d_uid.get<uint32_t>(), nnz, B.s);
    Scratch d_tmp2;
    if (!B.alloc(d_tmp2, scan2, "scan tmp")) return B.st;
    if (nnz > 0 && !B.ok(cub::DeviceScan::InclusiveSum(d_tmp2.p, scan2, heads, d_uid.get<uint32_t>(), nnz, B.s), "scan"))
        return B.st;

    // ---- 5. windows -> RowWindowOffset
    Scratch d_ustart, d_blocks, d_tmp3;
    if (!B.alloc(d_ustart, (size_t)(W + 1) * 4, "ustart") || !B.alloc(d_blocks, (size_t)(W + 1) * 4, "blocks") ||
        !B.ok(cudaMalloc((void **)&out.rwo, (size_t)(W + 1) * 4), "rwo"))
        return B.st;
    if (W > 0)
        window_kernel<<<grid_for(W), kThreads, 0, B.s>>>(d_sptr.get<int64_t>(), d_uid.get<uint32_t>(), W, rows, wh,
                                                         d_ustart.get<uint32_t>(), d_blocks.get<uint32_t>());
    if (!B.ok(cudaMemsetAsync(d_blocks.get<uint32_t>() + W, 0, 4, B.s), "memset")) return B.st;
    size_t scan3 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan3, d_blocks.get<uint32_t>(), out.rwo, W + 1, B.s);
    if (!B.alloc(d_tmp3, scan3, "scan tmp")) return B.st;
    if (!B.ok(cub::DeviceScan::ExclusiveSum(d_tmp3.p, scan3, d_blocks.get<uint32_t>(), out.rwo, W + 1, B.s), "scan"))
        return B.st;
    out.rwo_host.resize((size_t)W + 1);
    uint32_t total_u = 0;
    if (!B.ok(cudaMemcpyAsync(out.rwo_host.data(), out.rwo, (size_t)(W + 1) * 4, cudaMemcpyDeviceToHost, B.s), "D2H") ||
        (nnz > 0 && !B.ok(cudaMemcpyAsync(&total_u, d_uid.get<uint32_t>() + nnz - 1, 4, cudaMemcpyDeviceToHost, B.s), "D2H")) ||
        !B.ok(cudaStreamSynchronize(B.s), "sync"))
        return B.st;
    const int64_t NB = out.rwo_host[(size_t)W];
    if (NB * kWindow >= (int64_t)UINT32_MAX) return fail(ACCSPMM_ERR_UNSUPPORTED, "8*NB overflows u32 offsets");
    out.NB = NB;
    out.sum_U = total_u;

    // ---- 6. SparseAToB + TCLocalBit
    const size_t es = f16 ? 2 : 4;
    if (!B.ok(cudaMalloc((void **)&out.a2b, (size_t)(NB ? NB : 1) * 32), "a2b") ||
        // +2 words / +4 entries: the tcgen05 kernel bulk-copies 16-byte-aligned supersets
        !B.ok(cudaMalloc((void **)&out.bits, ((size_t)(NB ? NB : 1) * nwords + 2) * 8), "bits") ||
        !B.ok(cudaMalloc((void **)&out.tco, (size_t)(NB + 1 + 4) * 4), "tco") ||
        !B.ok(cudaMalloc(&out.vals, ((size_t)nnz + 16) * es), "vals"))
        return B.st;
    if (!B.ok(cudaMemsetAsync(out.a2b, 0xFF, (size_t)(NB ? NB : 1) * 32, B.s), "memset") ||  // kPadLane
        !B.ok(cudaMemsetAsync(out.bits, 0, ((size_t)(NB ? NB : 1) * nwords + 2) * 8, B.s), "memset") ||
        !B.ok(cudaMemsetAsync(out.tco, 0, (size_t)(NB + 1 + 4) * 4, B.s), "memset") ||
        !B.ok(cudaMemsetAsync(out.vals, 0, ((size_t)nnz + 16) * es, B.s), "memset"))
        return B.st;
    if (nnz > 0)
        fill_kernel<<<grid_for(nnz), kThreads, 0, B.s>>>(keys, d_uid.get<uint32_t>(), nnz, cbits, lw, d_ustart.get<uint32_t>(),
                                                         out.rwo, out.a2b,
                                                         reinterpret_cast<unsigned long long *>(out.bits));

    // ---- 7. TCOffset
    Scratch d_cnt, d_tmp4;
    if (!B.alloc(d_cnt, (size_t)(NB + 1) * 4, "popc")) return B.st;
    if (NB > 0)
        popc_kernel<<<grid_for(NB), kThreads, 0, B.s>>>(reinterpret_cast<const unsigned long long *>(out.bits), NB,
                                                        nwords, d_cnt.get<uint32_t>());
    if (!B.ok(cudaMemsetAsync(d_cnt.get<uint32_t>() + NB, 0, 4, B.s), "memset")) return B.st;
    size_t scan4 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan4, d_cnt.get<uint32_t>(), out.tco, NB + 1, B.s);
    if (!B.alloc(d_tmp4, scan4, "scan tmp")) return B.st;
    if (!B.ok(cub::DeviceScan::ExclusiveSum(d_tmp4.p, scan4, d_cnt.get<uint32_t>(), out.tco, NB + 1, B.s), "scan"))
        return B.st;

    // ---- 8. values in ascending bit order
    if (nnz > 0)
        values_kernel<<<grid_for(nnz), kThreads, 0, B.s>>>(keys, d_uid.get<uint32_t>(), vbits, nnz, cbits, lw,
                                                           d_ustart.get<uint32_t>(), out.rwo,
                                                           reinterpret_cast<const unsigned long long *>(out.bits),
                                                           out.tco, f16, out.vals);
    if (!B.ok(cudaGetLastError(), "launch") || !B.ok(cudaStreamSynchronize(B.s), "build")) return B.st;
    out.ms_build = std::chrono::duration<double, std::milli>(clk::now() - t_build).count();
    return ACCSPMM_OK;
}

void free_device_format(DeviceFormat &f)
{
    cudaFree(f.rwo);
    cudaFree(f.tco);
    cudaFree(f.a2b);
    cudaFree(f.bits);
    cudaFree(f.vals);
    f.rwo = f.tco = f.a2b = nullptr;
    f.bits = nullptr;
    f.vals = nullptr;
}

}  // namespace accspmm
