// Auxiliary device kernels: multi-GPU un-permute (K6), TF32 rounding and BitTCF
// decode test hooks.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../internal.hpp"

namespace accspmm {
namespace {

// C[orig_row[i]][:] = G[i][:]  (padding rows carry 0xFFFFFFFF and are skipped)
__global__ void unpermute_kernel(const float4 *__restrict__ G, const uint32_t *__restrict__ orig_row, int64_t n_rows,
                                 int64_t n4, float4 *__restrict__ C)
{
    const int64_t total = n_rows * n4;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n4, j = e - i * n4;
        const uint32_t o = __ldg(orig_row + i);
        if (o != 0xFFFFFFFFu) C[(int64_t)o * n4 + j] = __ldg(G + e);
    }
}

// Device SparseAToB relabelled to ORIGINAL column ids (permute_cols, hot columns R22): entry
// c' -> colorig[c'], padding lanes kept; with levels, lane 0 of every block also carries in bits
// 31..27 the bit length of its new id (the block's smallest: a window's columns ascend), i.e.
// the block's first column has new id < 2^level -- the hotness tag the kernel compares with the
// execute's hot-set size.
__global__ void relabel_cols_kernel(uint32_t *__restrict__ a2b, int64_t n, const uint32_t *__restrict__ colorig,
                                    int levels)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = a2b[e];
        if (c == kPadLane) continue;
        uint32_t o = __ldg(colorig + c);
        if (levels && (e & 7) == 0) o |= (uint32_t)(32 - __clz(c)) << kHotShift;
        a2b[e] = o;
    }
}

__global__ void round_tf32_kernel(const float *__restrict__ in, float *__restrict__ out, int64_t n)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(in[e]));
        out[e] = __uint_as_float(r);
    }
}

// tile[b][k] = value at bit k of TC block b: TCOffset[b] + popc(mask & (2^k - 1)), else 0
template <bool F16>
__global__ void decode_kernel(const uint64_t *__restrict__ bits, const uint32_t *__restrict__ tco,
                              const void *__restrict__ vals, int64_t NB, int nw, float *__restrict__ tiles)
{
    // tile b has nw*64 positions p = r*8 + lane (r < 8*nw); word p/64, bit p%64 (reading R20)
    const int64_t per = (int64_t)nw * 64;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NB * per; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / per;
        const int p = (int)(e - b * per);
        const int word = p >> 6, k = p & 63;
        const uint64_t m = __ldg(bits + b * nw + word);
        float v = 0.f;
        if ((m >> k) & 1ull) {
            uint32_t idx = __ldg(tco + b) + (uint32_t)__popcll(m & ((1ull << k) - 1ull));
            for (int j = 0; j < word; ++j) idx += (uint32_t)__popcll(__ldg(bits + b * nw + j));
            if (F16) v = __half2float(reinterpret_cast<const __half *>(vals)[idx]);
            else v = reinterpret_cast<const float *>(vals)[idx];
        }
        tiles[e] = v;
    }
}

// L2 read-bandwidth probe: every thread streams 128-bit L2-only loads (ld.global.cg) over
// an L2-resident buffer; the XOR of everything read is stored so nothing is elided.
template <int U>
__global__ void l2_read_kernel(const uint4 *__restrict__ buf, int64_t n16, int iters, uint32_t *__restrict__ sink)
{
    uint32_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int it = 0; it < iters; ++it) {
        int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; e + (U - 1) * stride < n16; e += U * stride) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(buf + e + u * stride));
#pragma unroll
            for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
        for (; e < n16; e += stride) {
            uint4 v;
            asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(buf + e));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (acc == 0x9E3779B9u) sink[0] = acc;  // practically never taken; keeps the loads live
}

// L2 read-bandwidth probe through the TMA engine (the SpMM kernel's B rows arrive this way):
// one thread per CTA streams CHUNK-byte bulk copies (cp.async.bulk global -> shared, mbarrier
// complete_tx) of the L2-resident buffer through an ST-stage shared-memory ring.
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int ST, int CHUNK>
__global__ void __launch_bounds__(32) l2_bulk_kernel(const uint8_t *__restrict__ buf, int64_t nchunks, int iters)
{
    extern __shared__ __align__(128) uint8_t ring[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(ring + ST * CHUNK);
    if (threadIdx.x != 0) return;
    for (int s = 0; s < ST; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(bar + s)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    uint32_t q = 0;  // copies issued so far; copy q uses stage q % ST
    auto wait = [&](uint32_t s, uint32_t parity) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "W_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra W_%=;\n\t}\n" ::"r"(smem_addr(bar + s)),
            "r"(parity)
            : "memory");
    };
    for (int it = 0; it < iters; ++it) {
        for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++q) {
            const uint32_t s = q % ST;
            if (q >= (uint32_t)ST) wait(s, ((q / ST) - 1u) & 1u);  // the stage's previous copy landed
            const uint32_t b = smem_addr(bar + s);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(CHUNK) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    smem_addr(ring + s * CHUNK)),
                "l"(buf + c * CHUNK), "r"(CHUNK), "r"(b)
                : "memory");
        }
    }
    for (uint32_t r = q > (uint32_t)ST ? q - ST : 0u; r < q; ++r) wait(r % ST, (r / ST) & 1u);  // drain
}

int grid_for(int64_t n, int threads)
{
    int64_t g = (n + threads - 1) / threads;
    return (int)(g < 148 * 32 ? (g < 1 ? 1 : g) : 148 * 32);
}

accspmm_status check_launch(const char *what)
{
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ACCSPMM_OK : fail(ACCSPMM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

accspmm_status launch_relabel_cols(uint32_t *a2b, int64_t n, const uint32_t *colorig, bool levels, void *stream)
{
    if (n == 0) return ACCSPMM_OK;
    int64_t grid = (n + 255) / 256;
    if (grid > 148 * 32) grid = 148 * 32;
    relabel_cols_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a2b, n, colorig, levels ? 1 : 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("relabel launch: ") + cudaGetErrorString(e));
    return ACCSPMM_OK;
}

accspmm_status launch_unpermute(const float *G, const uint32_t *orig_row, int64_t n_rows, int64_t N, float *C,
                                void *stream)
{
    const int64_t n4 = N / 4;
    unpermute_kernel<<<grid_for(n_rows * n4, 256), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float4 *>(G), orig_row, n_rows, n4, reinterpret_cast<float4 *>(C));
    return check_launch("unpermute launch");
}

accspmm_status probe_l2_read(int64_t bytes, int iters, double *gbs, int mode)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    void *buf = nullptr;
    uint32_t *sink = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaError_t e = cudaMalloc(&buf, (size_t)bytes);
    if (e == cudaSuccess) e = cudaMalloc((void **)&sink, 4);
    if (e == cudaSuccess) e = cudaMemset(buf, 0x5A, (size_t)bytes);
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    const int64_t n16 = bytes / 16;
    const uint4 *b16 = reinterpret_cast<const uint4 *>(buf);
    double best = 0.0;
    // the best of a few launch shapes / load depths (the probe must not under-state the peak)
    for (int cfg = 0; cfg < 4 && e == cudaSuccess && mode != 2; ++cfg) {
        const unsigned grid = (unsigned)sms * (cfg & 1 ? 8 : 4);
        const int threads = cfg & 1 ? 256 : 512;
        auto kern = cfg < 2 ? l2_read_kernel<4> : l2_read_kernel<8>;
        kern<<<grid, threads>>>(b16, n16, 2, sink);  // warm L2
        cudaEventRecord(e0);
        kern<<<grid, threads>>>(b16, n16, iters, sink);
        cudaEventRecord(e1);
        float ms = 0.f;
        e = cudaEventSynchronize(e1);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (e == cudaSuccess && ms > 0.f) best = std::max(best, (double)n16 * 16.0 * iters / (ms * 1e-3) / 1e9);
    }
    // TMA bulk copies (mode 0 or 2): the best of ring depths / chunk sizes / CTAs per SM
    for (int cfg = 0; cfg < 4 && e == cudaSuccess && mode != 1; ++cfg) {
        struct Shape { void (*k)(const uint8_t *, int64_t, int); int chunk, st, per_sm; };
        const Shape sh[4] = {{l2_bulk_kernel<4, 16384>, 16384, 4, 3}, {l2_bulk_kernel<8, 8192>, 8192, 8, 3},
                             {l2_bulk_kernel<4, 4096>, 4096, 4, 12}, {l2_bulk_kernel<8, 2048>, 2048, 8, 12}};
        const Shape &x = sh[cfg];
        const int smem = x.st * x.chunk + 128;
        e = cudaFuncSetAttribute(x.k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) break;
        const int64_t nchunks = bytes / x.chunk;
        const unsigned grid = (unsigned)(sms * x.per_sm);
        const uint8_t *b8 = reinterpret_cast<const uint8_t *>(buf);
        x.k<<<grid, 32, smem>>>(b8, nchunks, 2);  // warm L2
        cudaEventRecord(e0);
        x.k<<<grid, 32, smem>>>(b8, nchunks, iters);
        cudaEventRecord(e1);
        float ms = 0.f;
        e = cudaEventSynchronize(e1);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (e == cudaSuccess && ms > 0.f)
            best = std::max(best, (double)nchunks * x.chunk * iters / (ms * 1e-3) / 1e9);
    }
    cudaFree(buf);
    cudaFree(sink);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("L2 probe: ") + cudaGetErrorString(e));
    *gbs = best;
    return ACCSPMM_OK;
}

accspmm_status launch_round_tf32(const float *in, float *out, int64_t n, void *stream)
{
    round_tf32_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(in, out, n);
    return check_launch("round_tf32 launch");
}

accspmm_status launch_decode(const DevicePlan &p, float *tiles, void *stream)
{
    const int nw = p.wh / kWindow;
    const int64_t n = p.NB * 64 * nw;
    if (p.precision == ACCSPMM_FP16)
        decode_kernel<true><<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(p.bits, p.tco, p.vals, p.NB, nw, tiles);
    else
        decode_kernel<false><<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(p.bits, p.tco, p.vals, p.NB, nw, tiles);
    return check_launch("decode launch");
}

}  // namespace accspmm
