// Acc-SpMM runtime kernel for sm_100a (B200): C = A . B with A in BitTCF.
//
// What it computes follows PAPER.md §3.3-§3.5: every 8x8 TC block of a RowWindow
// is decoded from its u64 bitmap with the popcount rule of P:273 and
// multiplied on the tensor cores against the 8 gathered rows of B, with the
// operands swapped so the gathered B slice is the 16x8 left operand and the 8x8
// sparse tile the right operand of m16n8k8.  TF32 inputs with
// FP32 accumulation; an FP16 variant uses m16n8k8.f16 (BASELINE north_star).
//
// How it does it is designed for B200, not translated from Alg. 2:
//   * one warp owns one work unit of the sparsity-aware schedule:
//     a run of whole windows, or an even segment of one long window;
//   * the unit's compressed A stream (TCLocalBit, TCOffset, SparseAToB) is read
//     in 32-block chunks with coalesced 64/128-bit loads and staged in shared
//     memory; each block's values are cp.async'ed next to its B rows;
//   * B rows of each block are gathered with 16-byte cp.async (LDGSTS) into a
//     per-warp STAGES-deep shared-memory ring (the paper's double buffer, P:325-331,
//     generalised to an S-stage ring); padding lanes are zero-filled by the copy
//     engine (src-size 0) so B[0, :] never leaks;
//   * rows are XOR-swizzled at 16-byte granularity so the fragment loads are
//     bank-conflict free;
//   * B elements are rounded with cvt.rna.tf32.f32 at fragment load;
//   * the accumulator tile (8 window rows x FW features) lives in registers;
//     the epilogue stores C rows with st.global.cs (streaming, the .wt intent of
//     P:282) through the row permutation of the reordering;
//   * split windows write partial tiles to a workspace; the last-arriving
//     segment (atomic counter) sums them in segment order -- deterministic
//     cross-row write-back.
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdlib>

#include "../internal.hpp"

namespace accspmm {
namespace {

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src, uint32_t src_bytes)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint32_t tf32_rna(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1)
{
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0)
{
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(b0));
}

__device__ __forceinline__ void st_cs_v4(float *p, float a, float b, float c, float d)
{
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__device__ __forceinline__ void st_cs_v2(float *p, float a, float b)
{
    asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};\n" ::"l"(p), "f"(a), "f"(b) : "memory");
}

// ------------------------------------------------------------------ configuration

template <int FW, bool F16>
struct Cfg {
    static constexpr int ES = F16 ? 2 : 4;              // bytes per B element
    static constexpr int MT = FW / 16;                  // m16 tiles per warp tile
    static constexpr int ROW_BYTES = FW * ES;           // one gathered B row slice
    static constexpr int ROW_CHUNKS = ROW_BYTES / 16;   // 16-byte chunks per row
    static constexpr int CHUNKS = 8 * ROW_CHUNKS;       // chunks per TC block
    static constexpr int CP_ITERS = (CHUNKS + 31) / 32; // cp.async per lane per block
    static constexpr int LANE_BYTES = FW * ES / 8;      // bytes of one row a lane consumes
    static constexpr int VAL_WORDS = F16 ? 34 : 64;     // staged value words per block
    // XOR mask on the 16-byte chunk index of row r: makes the fragment loads
    // conflict-free (lanes of one 8-lane phase hit 8 distinct bank groups).
    __device__ static __forceinline__ int swz(int r)
    {
        if (!F16) {
            if (FW == 128) return r & 3;
            if (FW == 64) return (r & 1) | ((r & 2) << 1);
            if (FW == 32) return (r & 3) << 1;
            return r & 2;                                  // FW == 16
        } else {
            const int t = r >> 1;
            if (FW == 128) return (t & 1) | ((t & 2) << 1);
            if (FW == 64) return (t & 3) << 1;
            if (FW == 32) return (t & 1) << 1;
            return 0;                                      // FW == 16
        }
    }
};

template <int FW, bool F16, int STAGES>
struct WarpSmem {
    using C = Cfg<FW, F16>;
    struct Stage {
        alignas(16) uint8_t b[8 * C::ROW_BYTES];
        uint32_t val[C::VAL_WORDS];
        uint64_t mask;
        uint32_t voff;
        uint32_t pad;
    };
    uint32_t a2b[256];
    uint64_t mask[32];
    uint32_t tco[32];
    Stage st[STAGES];
};

struct KParams {
    const uint32_t *__restrict__ rwo;
    const uint32_t *__restrict__ tco;
    const uint32_t *__restrict__ a2b;
    const uint64_t *__restrict__ bits;
    const void *__restrict__ vals;
    const uint4 *__restrict__ units;
    const uint32_t *__restrict__ row_map;
    const void *__restrict__ B;
    float *__restrict__ C;
    float *__restrict__ ws;
    uint32_t *__restrict__ counters;
    int64_t N;
    int64_t rows;
    int64_t n_units;
    int32_t nslices;
};

// ------------------------------------------------------------------ the kernel

template <int FW, bool F16, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32) spmm_bittcf_kernel(const KParams p)
{
    using CF = Cfg<FW, F16>;
    using SM = WarpSmem<FW, F16, STAGES>;
    constexpr int MT = CF::MT;
    extern __shared__ __align__(128) uint8_t smem_raw[];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int slice = (int)(blockIdx.x % (unsigned)p.nslices);
    const int64_t u = (int64_t)(blockIdx.x / (unsigned)p.nslices) * WARPS + warp;
    if (u >= p.n_units) return;  // warp-uniform; no CTA-wide barrier is used below
    SM &sm = reinterpret_cast<SM *>(smem_raw)[warp];

    const uint4 ua = __ldg(p.units + 2 * u);
    const uint4 ub = __ldg(p.units + 2 * u + 1);
    const uint32_t w0 = ua.x, nw = ua.y, b0 = ua.z, b1 = ua.w;
    const bool split = ub.x != kNoSplit;
    const int64_t f0 = (int64_t)slice * FW;
    const uint32_t my_rwo = (uint32_t)lane <= nw ? __ldg(p.rwo + w0 + lane) : 0u;

    const int g = lane >> 2, t = lane & 3;
    float acc[MT][4];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;

    // ---- epilogue: whole window -> C rows 2t, 2t+1 of window (w0 + wi)
    auto store_window = [&](uint32_t wi) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int64_t lr = (int64_t)(w0 + wi) * 8 + 2 * t + s;
            if (lr < p.rows) {
                const int64_t orow = p.row_map ? (int64_t)__ldg(p.row_map + lr) : lr;
                float *dst = p.C + orow * p.N + f0 + g * (FW / 8);
                if constexpr (MT >= 2) {
#pragma unroll
                    for (int q = 0; q < MT / 2; ++q)
                        st_cs_v4(dst + 4 * q, acc[2 * q][s], acc[2 * q][2 + s], acc[2 * q + 1][s],
                                 acc[2 * q + 1][2 + s]);
                } else {
                    st_cs_v2(dst, acc[0][s], acc[0][2 + s]);
                }
            }
        }
#pragma unroll
        for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
    };

    uint32_t wi = 0;
    uint32_t wend = split ? b1 : __shfl_sync(0xffffffffu, my_rwo, 1);
    auto flush_empty = [&](uint32_t j) {
        while (!split && wi < nw && wend == j) {
            store_window(wi);
            ++wi;
            wend = __shfl_sync(0xffffffffu, my_rwo, (int)(wi < nw ? wi + 1 : nw));
        }
    };

    // ---- producer side of the ring: stage block i (relative to b0)
    const uint32_t nblk = b1 - b0;
    const char *Bbase = reinterpret_cast<const char *>(p.B);
    auto issue = [&](uint32_t i) {
        if (i < nblk) {
            const uint32_t b = b0 + i;
            const uint32_t cs = i & 31u;
            if (cs == 0) {  // stage the next 32 blocks of the compressed A stream (coalesced loads)
                const uint32_t cnt = min(32u, nblk - i);
                uint64_t m = 0;
                uint32_t o = 0;
                if ((uint32_t)lane < cnt) {
                    m = __ldg(p.bits + b + lane);
                    o = __ldg(p.tco + b + lane);
                }
                const uint4 *src4 = reinterpret_cast<const uint4 *>(p.a2b + (size_t)b * 8);
                uint4 x0 = make_uint4(0, 0, 0, 0), x1 = x0;
                if ((uint32_t)lane < 2 * cnt) x0 = __ldg(src4 + lane);
                if ((uint32_t)lane + 32 < 2 * cnt) x1 = __ldg(src4 + lane + 32);
                __syncwarp();
                sm.mask[lane] = m;
                sm.tco[lane] = o;
                reinterpret_cast<uint4 *>(sm.a2b)[lane] = x0;
                reinterpret_cast<uint4 *>(sm.a2b)[lane + 32] = x1;
                __syncwarp();
            }
            const uint64_t mask = sm.mask[cs];
            const uint32_t t0 = sm.tco[cs];
            const int cnt = __popcll(mask);
            uint64_t cm = mask | (mask >> 32);
            cm |= cm >> 16;
            cm |= cm >> 8;
            const uint32_t colmask = (uint32_t)cm & 0xFFu;  // condensed lanes present in the block
            auto &st = sm.st[i % STAGES];
            const uint32_t sb = smem_u32(st.b);
#pragma unroll
            for (int k = 0; k < CF::CP_ITERS; ++k) {
                const int q = lane + 32 * k;
                if (q < CF::CHUNKS) {
                    const int r = q / CF::ROW_CHUNKS, c = q % CF::ROW_CHUNKS;
                    const uint32_t col = sm.a2b[cs * 8 + r];
                    const bool v = (colmask >> r) & 1u;
                    const char *src = v ? Bbase + ((int64_t)col * p.N + f0) * CF::ES + c * 16 : Bbase;
                    cp_async16(sb + r * CF::ROW_BYTES + ((c ^ CF::swz(r)) * 16), src, v ? 16u : 0u);
                }
            }
            const uint32_t sv = smem_u32(st.val);
            if constexpr (!F16) {
                const float *vp = reinterpret_cast<const float *>(p.vals) + t0;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int e = lane + 32 * k;
                    cp_async4(sv + 4 * e, e < cnt ? (const void *)(vp + e) : p.vals, e < cnt ? 4u : 0u);
                }
            } else {
                const uint32_t ws0 = t0 >> 1;
                const int nwords = (int)(((t0 + (uint32_t)cnt + 1u) >> 1) - ws0);
                const uint32_t *vp = reinterpret_cast<const uint32_t *>(p.vals) + ws0;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int e = lane + 32 * k;
                    if (e < CF::VAL_WORDS)
                        cp_async4(sv + 4 * e, e < nwords ? (const void *)(vp + e) : p.vals, e < nwords ? 4u : 0u);
                }
            }
            if (lane == 0) {
                st.mask = mask;
                st.voff = t0 & 1u;
            }
        }
        cp_async_commit();
    };

    // ---- consumer side: decode + tensor-core MMA of block i
    auto consume = [&](uint32_t i) {
        auto &st = sm.st[i % STAGES];
        const uint64_t mask = st.mask;
        const uint8_t *sb = st.b;
        if constexpr (!F16) {
            // sparse operand (mma B fragment): b0 = A[g][t], b1 = A[g][t+4]
            const int k0 = g * 8 + t, k1 = k0 + 4;
            const uint64_t one = 1ull;
            const float *sv = reinterpret_cast<const float *>(st.val);
            const uint32_t bb0 = ((mask >> k0) & one) ? __float_as_uint(sv[__popcll(mask & ((one << k0) - one))]) : 0u;
            const uint32_t bb1 = ((mask >> k1) & one) ? __float_as_uint(sv[__popcll(mask & ((one << k1) - one))]) : 0u;
            const uint8_t *r0 = sb + t * CF::ROW_BYTES;
            const uint8_t *r1 = sb + (t + 4) * CF::ROW_BYTES;
            if constexpr (FW >= 32) {
#pragma unroll
                for (int j = 0; j < FW / 32; ++j) {
                    const int c = g * (FW / 32) + j;
                    const float4 x = *reinterpret_cast<const float4 *>(r0 + ((c ^ CF::swz(t)) * 16));
                    const float4 y = *reinterpret_cast<const float4 *>(r1 + ((c ^ CF::swz(t + 4)) * 16));
                    mma_tf32(acc[2 * j], tf32_rna(x.x), tf32_rna(x.y), tf32_rna(y.x), tf32_rna(y.y), bb0, bb1);
                    mma_tf32(acc[2 * j + 1], tf32_rna(x.z), tf32_rna(x.w), tf32_rna(y.z), tf32_rna(y.w), bb0, bb1);
                }
            } else {  // FW == 16: 2 floats per lane per row
                const int c = g >> 1, h = (g & 1) * 8;
                const float2 x = *reinterpret_cast<const float2 *>(r0 + ((c ^ CF::swz(t)) * 16) + h);
                const float2 y = *reinterpret_cast<const float2 *>(r1 + ((c ^ CF::swz(t + 4)) * 16) + h);
                mma_tf32(acc[0], tf32_rna(x.x), tf32_rna(x.y), tf32_rna(y.x), tf32_rna(y.y), bb0, bb1);
            }
        } else {
            // sparse operand: b0 = {A[g][2t], A[g][2t+1]} (adjacent bits)
            const int k0 = g * 8 + 2 * t;
            const uint64_t one = 1ull;
            const uint16_t *sv = reinterpret_cast<const uint16_t *>(st.val) + st.voff;
            const uint32_t lo = ((mask >> k0) & one) ? sv[__popcll(mask & ((one << k0) - one))] : 0u;
            const uint32_t hi = ((mask >> (k0 + 1)) & one) ? sv[__popcll(mask & ((one << (k0 + 1)) - one))] : 0u;
            const uint32_t bb0 = lo | (hi << 16);
            const int ra = 2 * t, rb = 2 * t + 1;
            const uint8_t *r0 = sb + ra * CF::ROW_BYTES;
            const uint8_t *r1 = sb + rb * CF::ROW_BYTES;
            if constexpr (FW >= 64) {
#pragma unroll
                for (int j = 0; j < FW / 64; ++j) {
                    const int c = g * (FW / 64) + j;
                    const uint4 x = *reinterpret_cast<const uint4 *>(r0 + ((c ^ CF::swz(ra)) * 16));
                    const uint4 y = *reinterpret_cast<const uint4 *>(r1 + ((c ^ CF::swz(rb)) * 16));
                    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        mma_f16(acc[4 * j + e], __byte_perm(xs[e], ys[e], 0x5410), __byte_perm(xs[e], ys[e], 0x7632),
                                bb0);
                }
            } else if constexpr (FW == 32) {
                const int c = g >> 1, h = (g & 1) * 8;
                const uint2 x = *reinterpret_cast<const uint2 *>(r0 + ((c ^ CF::swz(ra)) * 16) + h);
                const uint2 y = *reinterpret_cast<const uint2 *>(r1 + ((c ^ CF::swz(rb)) * 16) + h);
                mma_f16(acc[0], __byte_perm(x.x, y.x, 0x5410), __byte_perm(x.x, y.x, 0x7632), bb0);
                mma_f16(acc[1], __byte_perm(x.y, y.y, 0x5410), __byte_perm(x.y, y.y, 0x7632), bb0);
            } else {  // FW == 16
                const int c = g >> 2, h = (g & 3) * 4;
                const uint32_t x = *reinterpret_cast<const uint32_t *>(r0 + ((c ^ CF::swz(ra)) * 16) + h);
                const uint32_t y = *reinterpret_cast<const uint32_t *>(r1 + ((c ^ CF::swz(rb)) * 16) + h);
                mma_f16(acc[0], __byte_perm(x, y, 0x5410), __byte_perm(x, y, 0x7632), bb0);
            }
        }
    };

    // ---- the pipelined block loop
#pragma unroll
    for (int i = 0; i < STAGES - 1; ++i) issue((uint32_t)i);
    flush_empty(b0);
    for (uint32_t i = 0; i < nblk; ++i) {
        issue(i + STAGES - 1);
        cp_async_wait<STAGES - 1>();
        __syncwarp();
        consume(i);
        __syncwarp();
        if (!split && b0 + i + 1 == wend) {
            store_window(wi);
            ++wi;
            wend = __shfl_sync(0xffffffffu, my_rwo, (int)(wi < nw ? wi + 1 : nw));
            flush_empty(b0 + i + 1);
        }
    }
    cp_async_wait<0>();

    if (split) {
        // ---- cross-row write-back of a split window: partial -> workspace, last arriver reduces
        const uint32_t sid = ub.x, seg = ub.y, nseg = ub.z, slot = ub.w;
        float *tile = p.ws + ((int64_t)slot * p.nslices + slice) * (8 * FW);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            float *dst = tile + (2 * t + s) * FW + g * (FW / 8);
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                dst[2 * m] = acc[m][s];
                dst[2 * m + 1] = acc[m][2 + s];
            }
        }
        __threadfence();
        __syncwarp();
        uint32_t prev = 0;
        if (lane == 0) prev = atomicAdd(p.counters + (int64_t)sid * p.nslices + slice, 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        (void)seg;
        if (prev == nseg - 1) {
            __threadfence();
            const float *first = p.ws + ((int64_t)(slot - seg) * p.nslices + slice) * (8 * FW);
#pragma unroll
            for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
            for (uint32_t k = 0; k < nseg; ++k) {
                const float *src = first + (int64_t)k * p.nslices * (8 * FW);
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const float *row = src + (2 * t + s) * FW + g * (FW / 8);
#pragma unroll
                    for (int m = 0; m < MT; ++m) {
                        acc[m][s] += __ldcg(row + 2 * m);
                        acc[m][2 + s] += __ldcg(row + 2 * m + 1);
                    }
                }
            }
            store_window(0);
            if (lane == 0) p.counters[(int64_t)sid * p.nslices + slice] = 0u;  // re-arm for the next execute
        }
    }
}

// ------------------------------------------------------------------ launch

template <int FW, bool F16, int WARPS, int STAGES>
accspmm_status launch_cfg(const KParams &kp, int64_t n_units, cudaStream_t stream)
{
    using SM = WarpSmem<FW, F16, STAGES>;
    const size_t smem = sizeof(SM) * WARPS;
    auto kern = spmm_bittcf_kernel<FW, F16, WARPS, STAGES>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
        configured = true;
    }
    const int64_t groups = (n_units + WARPS - 1) / WARPS;
    const int64_t grid = groups * kp.nslices;
    if (grid > 0x7FFFFFFFll) return fail(ACCSPMM_ERR_UNSUPPORTED, "grid too large");
    kern<<<(unsigned)grid, WARPS * 32, smem, stream>>>(kp);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("spmm launch: ") + cudaGetErrorString(e));
    return ACCSPMM_OK;
}

int env_int(const char *name, int dflt)
{
    const char *s = std::getenv(name);
    return s ? std::atoi(s) : dflt;
}

template <int FW, bool F16>
accspmm_status launch_fw(const KParams &kp, int64_t n_units, cudaStream_t stream)
{
    // (warps per CTA, stages) variants; ACCSPMM_KCFG selects one for tuning.
    switch (env_int("ACCSPMM_KCFG", 0)) {
    case 1: return launch_cfg<FW, F16, 4, 3>(kp, n_units, stream);
    case 2: return launch_cfg<FW, F16, 4, 2>(kp, n_units, stream);
    case 3: return launch_cfg<FW, F16, 8, 2>(kp, n_units, stream);
    default: return launch_cfg<FW, F16, 4, 4>(kp, n_units, stream);
    }
}

}  // namespace

accspmm_status launch_spmm(const DevicePlan &d, const void *B, int64_t N, float *C, float *ws, uint32_t *counters,
                           void *stream)
{
    if (d.rows == 0) return ACCSPMM_OK;
    const int FW = N % 128 == 0 ? 128 : N % 64 == 0 ? 64 : N % 32 == 0 ? 32 : 16;
    KParams kp;
    kp.rwo = d.rwo;
    kp.tco = d.tco;
    kp.a2b = d.a2b;
    kp.bits = d.bits;
    kp.vals = d.vals;
    kp.units = reinterpret_cast<const uint4 *>(d.units);
    kp.row_map = d.row_map;
    kp.B = B;
    kp.C = C;
    kp.ws = ws;
    kp.counters = counters;
    kp.N = N;
    kp.rows = d.rows;
    kp.n_units = d.n_units;
    kp.nslices = (int32_t)(N / FW);
    cudaStream_t s = (cudaStream_t)stream;
    const bool f16 = d.precision == ACCSPMM_FP16;
    switch (FW) {
    case 128: return f16 ? launch_fw<128, true>(kp, d.n_units, s) : launch_fw<128, false>(kp, d.n_units, s);
    case 64: return f16 ? launch_fw<64, true>(kp, d.n_units, s) : launch_fw<64, false>(kp, d.n_units, s);
    case 32: return f16 ? launch_fw<32, true>(kp, d.n_units, s) : launch_fw<32, false>(kp, d.n_units, s);
    default: return f16 ? launch_fw<16, true>(kp, d.n_units, s) : launch_fw<16, false>(kp, d.n_units, s);
    }
}

}  // namespace accspmm
