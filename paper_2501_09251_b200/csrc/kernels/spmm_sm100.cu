// Acc-SpMM runtime kernel for sm_100a (B200): C = A . B with A in BitTCF.
//
// What it computes follows PAPER.md §3.3-§3.5: every 8x8 TC block of a RowWindow
// is decoded from its u64 bitmap with the popcount rule of P:273 and
// multiplied on the tensor cores against the 8 gathered rows of B, with the
// operands swapped so the gathered B slice is the 16x8 left operand and the 8x8
// sparse tile the right operand of m16n8k8.  TF32 inputs with
// FP32 accumulation; an FP16 variant uses m16n8k8.f16 (BASELINE north_star).
//
// How it does it is designed for B200, not translated from Alg. 2.  The
// default kernel is spmm_bittcf_g4_kernel:
//   * one warp = one CTA = one work unit of the sparsity-aware schedule (a run of
//     whole RowWindows or an even segment of a long window) x one FW-wide feature slice;
//     the grid is slice-major when N spans several slices;
//   * the unit's compressed A stream (TCLocalBit, TCOffset, SparseAToB) is staged 16 blocks
//     at a time by cp.async into a double-buffered shared-memory chunk;
//   * lane 0 gathers each block's 8 B rows with two TMA tile::gather4 requests into a
//     2-stage mbarrier ring (padding lanes ask for row -1: zero fill); the box is
//     32 bytes wider than the slice so the fragment loads are bank-conflict free;
//   * every lane decodes its two tile entries from the bitmap and loads their
//     values one block ahead; TF32 fragments come from LDS.128 (m16n8k4, or m16n8k8 at
//     FW <= 64), FP16 fragments from ldmatrix.trans; FP32 accumulators in registers;
//   * rho(B) (TF32 RNA) is applied once per execute by a pre-pass when B rows
//     are reused >= 32 times, else in registers after the LDS;
//   * the epilogue stores C rows with st.global.cs through the reordering permutation (Q12),
//     or, for the fused all-gather, into every rank's C; split windows go through a
//     workspace and the last-arriving segment sums the partials in segment order
//     (deterministic, Q18).
// spmm_bittcf_kernel (register-direct gather: each lane loads its fragment rows with
// 128-bit non-caching loads) and the other measured alternatives are compiled only into the
// variants build (-DACCSPMM_VARIANTS, libaccspmm_variants.so; ACCSPMM_KCFG selects them).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "../internal.hpp"

namespace accspmm {
namespace {

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// One lane of a converged warp (elect.sync).  Guarding a TMA issue with it instead of
// lane == 0 lets the compiler issue the uniform UTMALDG once, without the per-thread ELECT loop
// and divergent branch it emits for an arbitrary lane predicate (-~10 instructions per block).
__device__ __forceinline__ bool elect_one()
{
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}\n" : "=r"(pred));
    return pred != 0;
}

// A-stream staging copies.  No L2::cache_hint operand: with the constant-folded
// createpolicy value ptxas (12.9) emitted one LDGSTS of a large kernel with an uninitialised
// uniform descriptor register (desc[UR1], "illegal instruction" at run time); the policy
// argument is kept in the signature for the call sites and ignored.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint64_t)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src, uint64_t)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src, uint64_t)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

template <int BYTES>
struct Vec;
template <> struct Vec<16> { using T = uint4; };
template <> struct Vec<8> { using T = uint2; };
template <> struct Vec<4> { using T = uint32_t; };

__device__ __forceinline__ void ldg_nc(uint4 &v, const void *p, uint64_t pol)
{
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ldg_nc(uint2 &v, const void *p, uint64_t pol)
{
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;\n"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ldg_nc(uint32_t &v, const void *p, uint64_t pol)
{
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;\n" : "=r"(v) : "l"(p), "l"(pol));
}

// value loads with an L2 256-byte prefetch: a block's values are contiguous and the next
// blocks' follow, so one DRAM fetch serves several block steps (measurement variant)
__device__ __forceinline__ uint32_t ldg_pf256_u32(const void *p)
{
    uint32_t v;
    asm volatile("ld.global.nc.L2::256B.u32 %0, [%1];\n" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldg_pf256_u16(const void *p)
{
    unsigned short v;
    asm volatile("ld.global.nc.L2::256B.u16 %0, [%1];\n" : "=h"(v) : "l"(p));
    return (uint32_t)v;
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

// m16n8k4 TF32: A fragment = (row g, k t), (row g+8, k t) -> both come from one gathered row
__device__ __forceinline__ void mma_tf32_k4(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0)
{
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(b0));
}

__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0)
{
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(b0));
}

// ldmatrix .trans: the stored 8x8 b16 matrices are (gathered row k) x (8 consecutive features);
// thread (g, t) receives (k = 2t, 2t+1) of feature g packed -- the m16n8k8 A fragment
__device__ __forceinline__ void ldsm_x4_trans(uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3, uint32_t addr)
{
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_trans(uint32_t &r0, uint32_t &r1, uint32_t addr)
{
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void st_cs1(float *p, float a)
{
    asm volatile("st.global.cs.f32 [%0], %1;\n" ::"l"(p), "f"(a) : "memory");
}

__device__ __forceinline__ void st_cs(float *p, float a, float b, float c, float d)
{
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void st_cs(float *p, float a, float b)
{
    asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};\n" ::"l"(p), "f"(a), "f"(b) : "memory");
}

// ------------------------------------------------------------------ configuration

// Fragment geometry.  A lane (g = lane/4, t = lane%4) owns, for each of its two
// gathered rows (TF32: t and t+4; FP16: 2t and 2t+1), NV vectors of VW features;
// vector j covers features VW*(8j+g) .. +VW of the slice, so the 8 lanes sharing
// a row read (and later write) 8*VW contiguous features.  Feature slot f = VW*j+e
// of the lane is row (f&1 ? g+8 : g) of m16 tile mt = f>>1 (any bijection works
// for a product; this one makes both the loads and the stores coalesced).
template <int FW, bool F16>
struct Cfg {
    static constexpr int ES = F16 ? 2 : 4;
    static constexpr int MT = FW / 16;
    static constexpr int LPR = FW / 8;                                    // features per lane per row
    static constexpr int VB = LPR * ES >= 16 ? 16 : LPR * ES;             // vector bytes
    static constexpr int VW = VB / ES;                                    // features per vector
    static constexpr int NV = LPR / VW;                                   // vectors per row per lane
    using V = typename Vec<VB>::T;
};

constexpr int kChunk = 16;  // TC blocks per staged A-stream chunk

// X = extra TCOffset entries (value staging reads the TCOffset of the block after the chunk)
// NWD = occupancy words per block (1: the paper's 8-row windows; 2: 16-row windows, R20)
template <int X = 0, int NWD = 1>
struct ChunkSmemT {
    uint32_t a2b[kChunk * 8];
    uint64_t mask[kChunk * NWD];
    uint32_t tco[kChunk + X];
};
using ChunkSmem = ChunkSmemT<0>;

struct WarpSmem {
    ChunkSmem ch[2];
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
    const void *__restrict__ zrow;   // N zeros (the row padding lanes read)
    float *__restrict__ C;
    float *__restrict__ ws;
    uint32_t *__restrict__ counters;
    int64_t N;
    int64_t rows;
    int64_t n_units;
    int32_t nslices;
    int32_t Krows;
    int32_t slice_major;  // gather4 kernel: grid ordered slice-major (default when nslices > 1)
    // fused all-gather (accspmm_execute_allgather): every finished window row is also (only)
    // written to dst[0..ndst) -- full M x N matrices, local or peer memory -- at orig_map[row]
    int32_t ndst;
    // hot columns (R22): 255 = plan without hotness tags; else lane-0 SparseAToB entries carry a
    // tag in bits 31..27 and blocks with tag <= hot_lim gather with evict_last, the rest evict_first
    int32_t hot_lim;
    uint32_t id_mask;  // kHotIdMask for tagged plans, else all ones
    const uint32_t *__restrict__ orig_map;
    float *dst[kMaxGatherDst];
};

template <int FW, bool F16>
struct Frag {
    using CF = Cfg<FW, F16>;
    typename CF::V x[CF::NV];   // row rA (TF32: t, FP16: 2t)
    typename CF::V y[CF::NV];   // row rB (TF32: t+4, FP16: 2t+1)
    uint32_t b0, b1;            // decoded sparse-operand registers
};

template <int FW, bool F16>
__device__ __forceinline__ void mma_block(float (&acc)[Cfg<FW, F16>::MT][4], const Frag<FW, F16> &fr)
{
    using CF = Cfg<FW, F16>;
#pragma unroll
    for (int j = 0; j < CF::NV; ++j) {
        if constexpr (!F16) {
            if constexpr (CF::VW == 4) {
                const uint4 x = fr.x[j], y = fr.y[j];
                mma_tf32(acc[2 * j], x.x, x.y, y.x, y.y, fr.b0, fr.b1);
                mma_tf32(acc[2 * j + 1], x.z, x.w, y.z, y.w, fr.b0, fr.b1);
            } else {  // VW == 2 (FW == 16)
                const uint2 x = fr.x[j], y = fr.y[j];
                mma_tf32(acc[j], x.x, x.y, y.x, y.y, fr.b0, fr.b1);
            }
        } else {
            if constexpr (CF::VW == 8) {
                const uint4 x = fr.x[j], y = fr.y[j];
                const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    mma_f16(acc[4 * j + e], __byte_perm(xs[e], ys[e], 0x5410), __byte_perm(xs[e], ys[e], 0x7632),
                            fr.b0);
            } else if constexpr (CF::VW == 4) {
                const uint2 x = fr.x[j], y = fr.y[j];
                mma_f16(acc[2 * j], __byte_perm(x.x, y.x, 0x5410), __byte_perm(x.x, y.x, 0x7632), fr.b0);
                mma_f16(acc[2 * j + 1], __byte_perm(x.y, y.y, 0x5410), __byte_perm(x.y, y.y, 0x7632), fr.b0);
            } else {  // VW == 2
                const uint32_t x = fr.x[j], y = fr.y[j];
                mma_f16(acc[j], __byte_perm(x, y, 0x5410), __byte_perm(x, y, 0x7632), fr.b0);
            }
        }
    }
}

// Decode of one tile position: shifting the mask left by 63-k puts bit k on top;
// the popcount of the shifted word minus that top bit is popc(mask & (2^k - 1)).
__device__ __forceinline__ uint32_t tile_rank(uint64_t mask, uint32_t sh, bool &present)
{
    const uint64_t x = mask << sh;
    present = (int64_t)x < 0;
    return (uint32_t)__popcll(x) - (present ? 1u : 0u);
}

__device__ __forceinline__ uint32_t tf32_rna_bits(uint32_t x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(__uint_as_float(x)));
    return r;
}

// rho(B) applied to a loaded fragment (TF32 only; FP16 operands arrive already rounded)
template <int FW, bool F16>
__device__ __forceinline__ void round_frag(Frag<FW, F16> &fr)
{
    using CF = Cfg<FW, F16>;
    if constexpr (!F16) {
#pragma unroll
        for (int j = 0; j < CF::NV; ++j) {
            if constexpr (CF::VW == 4) {
                fr.x[j] = make_uint4(tf32_rna_bits(fr.x[j].x), tf32_rna_bits(fr.x[j].y), tf32_rna_bits(fr.x[j].z),
                                     tf32_rna_bits(fr.x[j].w));
                fr.y[j] = make_uint4(tf32_rna_bits(fr.y[j].x), tf32_rna_bits(fr.y[j].y), tf32_rna_bits(fr.y[j].z),
                                     tf32_rna_bits(fr.y[j].w));
            } else {
                fr.x[j] = make_uint2(tf32_rna_bits(fr.x[j].x), tf32_rna_bits(fr.x[j].y));
                fr.y[j] = make_uint2(tf32_rna_bits(fr.y[j].x), tf32_rna_bits(fr.y[j].y));
            }
        }
    }
}

// ------------------------------------------------------------------ the kernel

#ifdef ACCSPMM_VARIANTS
// Register-direct gather (variants build only): each lane loads its fragment rows with 128-bit
// non-caching loads; bound by the LSU data pipe, it lost to gather4 at every width.
template <int FW, bool F16, int WARPS, bool RND>
__global__ void __launch_bounds__(WARPS * 32) spmm_bittcf_kernel(const KParams p)
{
    using CF = Cfg<FW, F16>;
    using V = typename CF::V;
    constexpr int MT = CF::MT, NV = CF::NV, VW = CF::VW;
    __shared__ WarpSmem smem_all[WARPS];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int slice = (int)(blockIdx.x % (unsigned)p.nslices);
    const int64_t u = (int64_t)(blockIdx.x / (unsigned)p.nslices) * WARPS + warp;
    if (u >= p.n_units) return;  // warp-uniform; no CTA-wide barrier is used below
    WarpSmem &sm = smem_all[warp];
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();

    const uint4 ua = __ldg(p.units + 2 * u);
    const uint4 ub = __ldg(p.units + 2 * u + 1);
    const uint32_t w0 = ua.x, nw = ua.y, b0 = ua.z, b1 = ua.w;
    const bool split = ub.x != kNoSplit;
    const int64_t f0 = (int64_t)slice * FW;
    const uint32_t my_rwo = (uint32_t)lane <= nw ? __ldg(p.rwo + w0 + lane) : 0u;
    const uint32_t nblk = b1 - b0;

    const int g = lane >> 2, t = lane & 3;
    const int rA = F16 ? 2 * t : t, rB = F16 ? 2 * t + 1 : t + 4;
    const uint32_t sh0 = 63u - (uint32_t)(F16 ? g * 8 + 2 * t : g * 8 + t);
    const uint32_t sh1 = F16 ? sh0 - 1u : sh0 - 4u;
    // byte offset of this lane's vector j inside a gathered row slice
    const char *Bbase = reinterpret_cast<const char *>(p.B) + f0 * CF::ES + (int64_t)(VW * g) * CF::ES;
    const char *Zbase = reinterpret_cast<const char *>(p.zrow) + (int64_t)(VW * g) * CF::ES;
    const int64_t row_stride = p.N * CF::ES;

    // ---- A-stream chunk staging (cp.async, double buffered)
    auto issue_chunk = [&](uint32_t i) {  // blocks [b0+i, b0+i+32) -> buffer (i/32)&1
        if (i < nblk) {
            ChunkSmem &c = sm.ch[(i / kChunk) & 1];
            const uint32_t b = b0 + i;
            const uint32_t cnt = min((uint32_t)kChunk, nblk - i);
            if ((uint32_t)lane < cnt) {
                cp_async8(smem_u32(&c.mask[lane]), p.bits + b + lane, pol_stream);
                cp_async4(smem_u32(&c.tco[lane]), p.tco + b + lane, pol_stream);
            }
            const uint4 *src4 = reinterpret_cast<const uint4 *>(p.a2b + (size_t)b * 8);
            if ((uint32_t)lane < 2 * cnt) cp_async16(smem_u32(&c.a2b[4 * lane]), src4 + lane, pol_stream);
            if ((uint32_t)lane + 32 < 2 * cnt) cp_async16(smem_u32(&c.a2b[4 * (lane + 32)]), src4 + lane + 32, pol_stream);
        }
        cp_async_commit();
    };

    // ---- gather + decode of block i (relative to b0) into a register fragment
    auto load_block = [&](Frag<FW, F16> &fr, uint32_t i) {
        if ((i & (kChunk - 1u)) == 0) {  // chunk boundary: this chunk must have landed; prefetch the next one
            cp_async_wait_all();
            __syncwarp();
            issue_chunk(i + kChunk);
        }
        const ChunkSmem &c = sm.ch[(i / kChunk) & 1];
        const uint32_t cs = i & (kChunk - 1u);
        const uint64_t mask = c.mask[cs];
        const uint32_t t0 = c.tco[cs];
        uint64_t cm = mask | (mask >> 32);
        cm |= cm >> 16;
        cm |= cm >> 8;  // low byte: condensed lanes present in the block
        const bool va = (cm >> rA) & 1u, vb = (cm >> rB) & 1u;
        const char *pa = va ? Bbase + (int64_t)c.a2b[cs * 8 + rA] * row_stride : Zbase;
        const char *pb = vb ? Bbase + (int64_t)c.a2b[cs * 8 + rB] * row_stride : Zbase;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            ldg_nc(fr.x[j], pa + j * 8 * CF::VB, pol_keep);
            ldg_nc(fr.y[j], pb + j * 8 * CF::VB, pol_keep);
        }
        // sparse operand: value index = TCOffset + popc(mask & (2^k - 1))
        bool p0, p1;
        const uint32_t i0 = t0 + tile_rank(mask, sh0, p0);
        const uint32_t i1 = t0 + tile_rank(mask, sh1, p1);
        if constexpr (!F16) {
            const float *vp = reinterpret_cast<const float *>(p.vals);
            fr.b0 = p0 ? __float_as_uint(__ldg(vp + i0)) : 0u;
            fr.b1 = p1 ? __float_as_uint(__ldg(vp + i1)) : 0u;
        } else {
            const unsigned short *vp = reinterpret_cast<const unsigned short *>(p.vals);
            const uint32_t lo = p0 ? (uint32_t)__ldg(vp + i0) : 0u;
            const uint32_t hi = p1 ? (uint32_t)__ldg(vp + i1) : 0u;
            fr.b0 = lo | (hi << 16);
            fr.b1 = 0u;
        }
    };

    float acc[MT][4];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;

    // ---- epilogue: whole window -> C rows 2t, 2t+1 of window (w0 + wi)
    auto store_rows = [&](float *base, int64_t ld, int64_t lr0, bool remap) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int64_t lr = lr0 + 2 * t + s;
            if (!remap || lr < p.rows) {
                const int64_t orow = remap ? (p.row_map ? (int64_t)__ldg(p.row_map + lr) : lr) : (2 * t + s);
                float *dst = base + orow * ld + VW * g;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    float *d = dst + 8 * VW * j;
                    if constexpr (VW == 2) {
                        st_cs(d, acc[j][s], acc[j][2 + s]);
                    } else {
#pragma unroll
                        for (int q = 0; q < VW / 4; ++q) {
                            const int m0 = (VW / 2) * j + 2 * q;
                            st_cs(d + 4 * q, acc[m0][s], acc[m0][2 + s], acc[m0 + 1][s], acc[m0 + 1][2 + s]);
                        }
                    }
                }
            }
        }
    };
    auto store_window = [&](uint32_t wi) {
        store_rows(p.C + f0, p.N, (int64_t)(w0 + wi) * 8, true);
#pragma unroll
        for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
    };

    uint32_t wi = 0;
    uint32_t wend = split ? b1 : __shfl_sync(0xffffffffu, my_rwo, 1);
    auto after_block = [&](uint32_t jnext) {  // jnext = absolute index of the next block
        while (!split && wi < nw && wend == jnext) {
            store_window(wi);
            ++wi;
            wend = __shfl_sync(0xffffffffu, my_rwo, (int)(wi < nw ? wi + 1 : nw));
        }
    };

    // ---- pipelined block loop: two register fragments in flight per warp
    issue_chunk(0);
    after_block(b0);  // leading empty windows
    Frag<FW, F16> fa, fb;
    if (nblk > 0) load_block(fa, 0);
    if (nblk > 1) load_block(fb, 1);
    for (uint32_t i = 0; i < nblk; i += 2) {
        if constexpr (RND) round_frag<FW, F16>(fa);
        mma_block<FW, F16>(acc, fa);
        after_block(b0 + i + 1);
        if (i + 2 < nblk) load_block(fa, i + 2);
        if (i + 1 < nblk) {
            if constexpr (RND) round_frag<FW, F16>(fb);
            mma_block<FW, F16>(acc, fb);
            after_block(b0 + i + 2);
            if (i + 3 < nblk) load_block(fb, i + 3);
        }
    }
    cp_async_wait_all();

    if (split) {
        // ---- cross-row write-back of a split window: partial -> workspace, last arriver reduces
        const uint32_t sid = ub.x, seg = ub.y, nseg = ub.z, slot = ub.w;
        float *tile = p.ws + ((int64_t)slot * p.nslices + slice) * (8 * FW);
        store_rows(tile, FW, 0, false);
        __threadfence();
        __syncwarp();
        uint32_t prev = 0;
        if (lane == 0) prev = atomicAdd(p.counters + (int64_t)sid * p.nslices + slice, 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == nseg - 1) {
            __threadfence();
            const float *first = p.ws + ((int64_t)(slot - seg) * p.nslices + slice) * (8 * FW);
#pragma unroll
            for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
            for (uint32_t k = 0; k < nseg; ++k) {
                const float *src = first + (int64_t)k * p.nslices * (8 * FW);
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const float *row = src + (2 * t + s) * FW + VW * g;
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
#pragma unroll
                        for (int e = 0; e < VW; e += 2) {
                            const int m = (VW / 2) * j + (e >> 1);
                            const float2 v = __ldcg(reinterpret_cast<const float2 *>(row + 8 * VW * j + e));
                            acc[m][s] += v.x;
                            acc[m][2 + s] += v.y;
                        }
                    }
                }
            }
            store_window(0);
            if (lane == 0) p.counters[(int64_t)sid * p.nslices + slice] = 0u;  // re-arm for the next execute
        }
    }
}
#endif  // ACCSPMM_VARIANTS


// ================================================================== mbarrier / TMA helpers

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}\n" ::"r"(bar), "r"(phase), "r"(0x989680)
        : "memory");
}

// WT = 0: try_wait with a suspend-time hint (the default); 1: try_wait without a hint;
// 2: test_wait spin (never suspends) -- measurement variants of the stage wait
template <int WT>
__device__ __forceinline__ void mbar_wait_t(uint32_t bar, uint32_t phase)
{
    if constexpr (WT == 0) {
        mbar_wait(bar, phase);
    } else if constexpr (WT == 1) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@P1 bra DONE_%=;\n\t"
            "bra WAIT_%=;\n\t"
            "DONE_%=:\n\t}\n" ::"r"(bar), "r"(phase)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "WAIT_%=:\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@P1 bra DONE_%=;\n\t"
            "bra WAIT_%=;\n\t"
            "DONE_%=:\n\t}\n" ::"r"(bar), "r"(phase)
            : "memory");
    }
}

// ================================================================== v4: TMA gather4
//
// v3 issues 9 bulk copies per TC block and becomes TMA-request bound (~10 SM
// cycles per request).  v4 uses the sm_100 tensor gather:
// cp.async.bulk.tensor.2d.tile::gather4 brings 4 arbitrary B rows (box FW+8
// elements wide) per instruction, so a block costs 2 gathers + 1 bulk copy of its
// values.  Padding lanes ask for row K, which the TMA zero-fills.
// The box is 8 elements wider than the slice so consecutive gathered rows land
// 32 B (TF32) / 16 B (FP16) off a 128-byte bank period: the fragment LDS of each
// 8-lane phase then touches 8 distinct bank groups.  Gather 1 carries the rows of
// fragment x (TF32 rows 0-3, FP16 rows 0,2,4,6), gather 2 those of fragment y.

// B3 (TF32 only): B is gathered from its 3-byte TF32 image (DESIGN.md §6 "B3"): per feature
// slice, FW high halves (bits 31..16 of rho(b)) then FW bytes of bits 15..8 -- lossless, since
// rho(b) has bits 12..0 zero -- so a gathered row is 3*FW bytes instead of 4*FW.
template <int FW, bool F16, bool B3 = false>
struct G4Cfg {
    using CF = Cfg<FW, F16>;
    static_assert(!B3 || (!F16 && FW >= 64), "B3: TF32 slices of 64 or 128 features");
    // box width: gathered rows then sit 32 B off a 128-byte bank period, so the fragment loads
    // of one phase (LDS.128: 4 rows x 2 column groups; B3 LDS.64: 4 rows x 4) hit distinct banks
    static constexpr int RS = B3 ? 3 * FW + 32 : (FW + 32 / CF::ES) * CF::ES;  // gathered row stride
    static constexpr int BOXE = B3 ? RS / 2 : RS / CF::ES;  // box width in tensor-map elements
    static constexpr int GRP = (4 * RS + 127) / 128 * 128;   // one gather4 (4 rows), 128-aligned
    static constexpr int STAGE_AL = 2 * GRP;
};

// VST > 0: each chunk's value range (up to VST values) is staged by one bulk copy a chunk
// ahead; the chunk metadata is then triple buffered (chunk c + 2 is in flight while the
// values of chunk c + 1 are copied).  CX = extra TCOffset slots per chunk.
// Layout note (measured): the stage mbarriers sit 16-byte aligned right after
// the chunk metadata; a layout that put them at 8 mod 16 behind other fields ran the default
// kernel 2.2x slower (5.55 vs 2.54 ms on the Reddit-shaped bench) with identical SASS apart
// from the shared-memory offsets.
// BS = barrier stride in 8-byte words (1: packed; 2: one 16-byte slot per stage barrier;
// 16: one 128-byte line each -- measurement variants)
template <int FW, bool F16, int STAGES, int VST = 0, int CX = (VST ? 4 : 0), bool B3 = false, int BS = 1,
          int NWD = 1>
struct G4WarpSmem {
    alignas(128) uint8_t stage[STAGES][G4Cfg<FW, F16, B3>::STAGE_AL];
    ChunkSmemT<CX, NWD> ch[VST ? 3 : 2];
    alignas(BS >= 16 ? 128 : 16) uint64_t bar[STAGES * BS];
    uint64_t vbar[2];
    uint32_t vlo[2];  // first staged value index per buffer (0xFFFFFFFF: over VST, values from L2)
    alignas(16) uint8_t vals[VST ? 2 : 1][VST ? VST * (F16 ? 2 : 4) : 16];
};
// measurement variants: the same layout with PAD more bytes of per-CTA shared-memory footprint
template <typename Base, int PAD>
struct G4Padded : Base {
    uint8_t pad[PAD];
};
// the same fields with the stage barriers at the head of the warp's area (BS = 0 in the kernel)
template <int FW, bool F16, int STAGES, int VST = 0, int CX = (VST ? 4 : 0), bool B3 = false>
struct G4WarpSmemHead {
    alignas(128) uint64_t bar[STAGES];
    uint64_t vbar[2];
    uint32_t vlo[2];
    alignas(128) uint8_t stage[STAGES][G4Cfg<FW, F16, B3>::STAGE_AL];
    ChunkSmemT<CX> ch[VST ? 3 : 2];
    alignas(16) uint8_t vals[VST ? 2 : 1][VST ? VST * (F16 ? 2 : 4) : 16];
};
template <int FW, bool F16, int STAGES, int VST, int CX, bool B3, int BS, int NWD = 1, int PAD = 0>
using G4Smem = std::conditional_t<
    BS == 0, G4WarpSmemHead<FW, F16, STAGES, VST, CX, B3>,
    std::conditional_t<PAD == 0, G4WarpSmem<FW, F16, STAGES, VST, CX, B3, BS, NWD>,
                       G4Padded<G4WarpSmem<FW, F16, STAGES, VST, CX, B3, BS, NWD>, (PAD > 0 ? PAD : 1)>>>;
static_assert(sizeof(ChunkSmemT<0>) % 16 == 0 && sizeof(ChunkSmemT<4>) % 16 == 0 && sizeof(ChunkSmemT<0, 2>) % 16 == 0,
              "chunk alignment (cp.async 16 B into a2b)");

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap *map, int32_t col, int32_t r0, int32_t r1,
                                            int32_t r2, int32_t r3, uint32_t bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar),
          "l"(pol)
        : "memory");
}

// Tensor maps of B: with nmaps > 1, map s covers exactly feature slice s (base B + s*FW,
// width FW), so the box's extra columns fall outside the tensor and are zero-filled
// without L2 traffic; with nmaps == 1 one map spans all N columns (N == FW, or more
// slices than maps: the extra columns of a box are then real reads of the next slice).
constexpr int kMaxSliceMaps = 8;
template <int NM>
struct G4MapsT {
    CUtensorMap m[NM];
};
using G4Maps = G4MapsT<kMaxSliceMaps>;
inline int map_count(const KParams &kp) { return kp.nslices > 1 && kp.nslices <= kMaxSliceMaps ? kp.nslices : 1; }

template <int FW, bool F16, int WARPS, int STAGES, bool RND, int MINB = 1, int NM = 1, bool LDSM_ = false,
          bool K8 = false, int VD = 1, int PF256 = 0, int VST = 0, bool HYB = false, int CX = (VST ? 4 : 0),
          bool B3 = false, bool DEC64 = false, int EL = 1, bool HT = true, bool PIN = false, bool DYN = false,
          int BS = 1, int WT = 0, int WH = 8, bool L64 = false, int PAD = 0>
__global__ void __launch_bounds__(WARPS * 32, MINB)
    spmm_bittcf_g4_kernel(const KParams p, const __grid_constant__ G4MapsT<NM> maps)
{
    // HYB: hybrid gather -- odd blocks (stage 1) are gathered by cp.async from every lane (LSU
    // path) into the exact layout the TMA gives even blocks (stage 0), so the two request
    // engines share the request-bound regimes (FP16, narrow N)
    static_assert(!HYB || (STAGES == 2 && WARPS == 1), "hybrid gather: default ring only");
    static_assert(VST == 0 || (STAGES == 2 && VD == 1), "value staging: default ring only");
    // LDSM (FP16 only): A fragments by ldmatrix.trans straight from the gathered rows (no
    // PRMT packing); gather y is fetched 8 columns early so its rows sit 16 B off gather x's
    // and the 8 row addresses of every ldmatrix phase hit 8 distinct bank groups.  The
    // accumulator layout is then m16 tile mt = features 16mt .. 16mt+15 (epilogue below).
    constexpr bool LDSM = LDSM_ && F16;
    // WH = 16 (reading R20 on the mma.sync kernel): a block is a 16 x 8 tile (two occupancy
    // words); each gathered row feeds NH = 2 accumulator halves (window rows 0-7 and 8-15), so
    // the two gathers of a block serve twice the rows.  Default ring and value path only.
    constexpr int NH = WH / 8;
    // L64 (TF32, FW >= 32): one m16n8k8 per m16 tile with its four A registers loaded by two
    // LDS.64 (row t from gather x, row t + 4 from gather y) -- no register moves (the LDS.128
    // form needs 3 MOVs per k8 MMA) and half the tensor-pipe cycles of two m16n8k4.  Gathered
    // rows are FW + 4 elements apart (RS = 16 mod 128) and lane g's 8-byte piece tau of 32-feature
    // chunk j sits at slot (g & 1) + 8 ((g >> 1) & 1) + 4 (g >> 2) + 2 tau, so the 16 lanes of each
    // LDS.64 phase (4 rows x 4 pieces) hit 16 distinct 8-byte bank pairs.
    static_assert(!L64 || (!F16 && FW >= 32 && !B3 && !HYB && VST == 0 && !LDSM_), "L64: TF32 slices >= 32");
    static_assert(WH == 8 || (WH == 16 && STAGES == 2 && VD == 1 && PF256 == 0 && VST == 0 && !HYB && !B3 &&
                              !DEC64 && !DYN && !HT && BS >= 1),
                  "16-row windows: the default kernel configuration");
    constexpr int CH = kChunk;  // blocks per staged chunk
    using CF = Cfg<FW, F16>;
    using GC = G4Cfg<FW, F16, B3>;
    using SM = G4Smem<FW, F16, STAGES, VST, CX, B3, BS, WH / 8, PAD>;
    constexpr int RS = L64 ? (FW + 4) * 4 : GC::RS;
    static_assert(!L64 || RS % 128 == 16, "L64 row stride");
    static_assert(!B3 || (!RND && !HYB && VST == 0 && !LDSM_), "B3: pre-rounded B, default ring");
    static_assert(VST == 0 || CX >= 1, "value staging reads the TCOffset after the chunk");
    using SMB = G4Smem<FW, F16, STAGES, VST, CX, B3, BS, WH / 8>;  // the layout without padding
    static_assert(offsetof(SMB, bar) % 16 == 0, "stage mbarriers 16-byte aligned (measured: 2.2x slower otherwise)");
    constexpr int BSTR = BS == 0 ? 1 : BS;  // barrier stride (BS = 0: packed, at the head)
    using V = typename CF::V;
    constexpr int MT = CF::MT;
    // epilogue geometry: lane g owns NV vectors of VW features, vector j = features VW*(8j+g)..
    // (B3: 8-feature groups 64j + 8g .. +7, the units of its LDS.128 of high halves)
    constexpr int VW = B3 ? 8 : CF::VW, NV = B3 ? FW / 64 : CF::NV;
    constexpr int NCB = VST ? 3 : 2;  // chunk metadata buffers
    extern __shared__ __align__(128) uint8_t smem_raw[];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // slice-fastest order: the slices of a unit run together and share its A stream in L2;
    // slice-major (p.slice_major): one feature slice of B at a time is the L2 working set
    const unsigned ngrp = (unsigned)((p.n_units + WARPS - 1) / WARPS);
    const int slice = p.slice_major ? (int)(blockIdx.x / ngrp) : (int)(blockIdx.x % (unsigned)p.nslices);
    const int64_t u = (int64_t)(p.slice_major ? blockIdx.x % ngrp : blockIdx.x / (unsigned)p.nslices) * WARPS + warp;
    if (u >= p.n_units) return;  // warp-uniform; only warp-scoped synchronisation below
    SM &sm = reinterpret_cast<SM *>(smem_raw)[warp];
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    if (lane == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.m[NM > 1 ? slice : 0]))
                     : "memory");
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(&sm.bar[s * BSTR]), (HYB && s == 1) ? 32 : 1);
        if constexpr (VST > 0) {
            mbar_init(smem_u32(&sm.vbar[0]), 1);
            mbar_init(smem_u32(&sm.vbar[1]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();

    const uint4 ua = __ldg(p.units + 2 * u);
    const uint4 ub = __ldg(p.units + 2 * u + 1);
    const uint32_t w0 = ua.x, nw = ua.y, b0 = ua.z, b1 = ua.w;
    const bool split = ub.x != kNoSplit;
    const int64_t f0 = (int64_t)slice * FW;
    const uint32_t my_rwo = (uint32_t)lane <= nw ? __ldg(p.rwo + w0 + lane) : 0u;
    const uint32_t nblk = b1 - b0;
    const int g = lane >> 2, t = lane & 3;
    // this lane's two positions of the 8x8 tile (the mma B fragment), as shift amounts 63-k
    const int k0 = F16 ? g * 8 + 2 * t : g * 8 + t;
    const int k1 = F16 ? k0 + 1 : k0 + 4;
    const uint32_t sh0 = 63u - (uint32_t)k0, sh1 = 63u - (uint32_t)k1;
    // 32-bit decode (default): k0 < k1 lie in one 32-bit half of the mask (row g's byte), so
    // rank(k0) = popc(lo & m_lo) + popc(hi & m_hi) with lane-constant masks, and rank(k1) adds
    // the popcount of the DK bits k0 .. k1-1 (DEC64 = the 64-bit shift form, tile_rank)
    constexpr uint32_t DK = F16 ? 1u : 4u;
    const uint32_t hw = (uint32_t)k0 >> 5, p0w = (uint32_t)k0 & 31u;
    const uint32_t below = (1u << p0w) - 1u;
    uint32_t m_lo = hw ? 0xFFFFFFFFu : below, m_hi = hw ? below : 0u;
    // PIN: keep the lane constants and the value base in registers (an empty asm hides their
    // derivation, so the compiler cannot rematerialise them inside the block loop)
    const char *vals_base = reinterpret_cast<const char *>(p.vals);
    // this lane's fragment offset in a stage (L64: row t, slot of piece tau = 0)
    const uint32_t l64_slot = (uint32_t)((g & 1) + 8 * ((g >> 1) & 1) + 4 * (g >> 2));
    uint32_t frag_off = L64 ? (uint32_t)(t * RS + 8 * l64_slot) : (uint32_t)(t * GC::RS + CF::VB * g);
    if constexpr (PIN) {
        asm volatile("" : "+r"(m_lo), "+r"(m_hi), "+r"(frag_off));
        asm volatile("" : "+l"(vals_base));
    }

    auto issue_chunk = [&](uint32_t i) {
        if (i < nblk) {
            auto &c = sm.ch[(i / CH) % NCB];
            const uint32_t b = b0 + i;
            const uint32_t cnt = min((uint32_t)CH, nblk - i);
            if ((uint32_t)lane < cnt) {
                if constexpr (NH == 1)
                    cp_async8(smem_u32(&c.mask[lane]), p.bits + b + lane, pol_stream);
                else
                    cp_async16(smem_u32(&c.mask[2 * lane]), p.bits + 2 * ((size_t)b + lane), pol_stream);
                cp_async4(smem_u32(&c.tco[lane]), p.tco + b + lane, pol_stream);
            }
            if (VST > 0 && (uint32_t)lane == cnt) cp_async4(smem_u32(&c.tco[lane]), p.tco + b + lane, pol_stream);
            const uint4 *src4 = reinterpret_cast<const uint4 *>(p.a2b + (size_t)b * 8);
            if ((uint32_t)lane < 2 * cnt) cp_async16(smem_u32(&c.a2b[4 * lane]), src4 + lane, pol_stream);
            if (2 * CH > 32 && (uint32_t)lane + 32 < 2 * cnt)
                cp_async16(smem_u32(&c.a2b[4 * (lane + 32)]), src4 + lane + 32, pol_stream);
        }
        cp_async_commit();
    };
    // Value registers of the blocks in flight: decoded and loaded VD blocks ahead of use (a
    // VR-slot register ring).  A bulk L2 prefetch of each chunk's value range and staging
    // values through shared memory were measured and lost.
    static_assert(VD == 1 || VD == 2, "value distance");
    // DYN (deep ring, STAGES > 2): values are loaded with the TMA of their block, STAGES - 1
    // blocks ahead, so up to STAGES value slots are live
    static_assert(!DYN || (STAGES > 2 && STAGES <= 4 && VST == 0 && !HYB), "deep ring: 3 or 4 stages");
    constexpr int VR = DYN ? 4 : VD == 1 ? 2 : 4;
    uint32_t vb0[VR], vb1[VR];
    uint32_t vc0[NH == 2 ? VR : 1], vc1[NH == 2 ? VR : 1];  // window rows 8-15 (WH = 16)
    constexpr int SM1 = NH == 2 ? VR - 1 : 0;                // their slot mask
    // PF256 == 3 (measurement variant): the block's value run is loaded by one coalesced warp
    // load (lane L: value tco + L, and tco + 32 + L when the block holds more than 32); the
    // lane's two entries are picked by shuffles at consume time.  vix = packed local indices
    // (bits 0-5, 6-11), presence (12, 13) and "more than 32 values" (14).
    uint32_t vix[PF256 == 3 ? VR : 1];

    // ---- lane 0 (VST): bulk copy of chunk c's value range (16-byte-aligned superset; the
    // value allocation carries 16 elements of padding) into value buffer c & 1
    auto issue_vals = [&](uint32_t c) {
        if constexpr (VST > 0) {
            if (lane != 0 || c * CH >= nblk) return;
            constexpr uint32_t AL = 16 / CF::ES;  // elements per 16 bytes
            const auto &m = sm.ch[c % NCB];
            const uint32_t cnt = min((uint32_t)CH, nblk - c * CH);
            const uint32_t v_lo = m.tco[0] & ~(AL - 1u), v_hi = (m.tco[cnt] + AL - 1u) & ~(AL - 1u);
            const uint32_t bar = smem_u32(&sm.vbar[c & 1]);
            if (v_hi - v_lo <= (uint32_t)VST) {
                sm.vlo[c & 1] = v_lo;
                mbar_arrive_expect_tx(bar, (v_hi - v_lo) * CF::ES);
                if (v_hi > v_lo)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                            smem_u32(sm.vals[c & 1])),
                        "l"(reinterpret_cast<const char *>(p.vals) + (size_t)v_lo * CF::ES), "r"((v_hi - v_lo) * CF::ES),
                        "r"(bar)
                        : "memory");
            } else {
                sm.vlo[c & 1] = 0xFFFFFFFFu;
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
            }
        }
    };
    // ---- every lane: decode this lane's two tile entries of block j, load values
    auto value_load = [&](uint32_t j, int slot) {
        const auto &c = sm.ch[(j / CH) % NCB];
        const uint32_t cs = j & (CH - 1u);
        const uint64_t mask = c.mask[cs * NH];
        const uint32_t t0 = c.tco[cs];
        bool p0, p1;
        uint32_t i0, i1;
        if constexpr (DEC64) {
            i0 = t0 + tile_rank(mask, sh0, p0);
            i1 = t0 + tile_rank(mask, sh1, p1);
        } else {
            const uint32_t lo = (uint32_t)mask, hi = (uint32_t)(mask >> 32);
            const uint32_t r = (hw ? hi : lo) >> p0w;  // bit 0 = position k0, bit DK = k1
            p0 = (r & 1u) != 0u;
            p1 = ((r >> DK) & 1u) != 0u;
            i0 = t0 + (uint32_t)__popc(lo & m_lo) + (uint32_t)__popc(hi & m_hi);
            i1 = i0 + (uint32_t)__popc(r & ((1u << DK) - 1u));
        }
        if constexpr (PF256 == 3) {
            const uint32_t lo = (uint32_t)mask, hi = (uint32_t)(mask >> 32);
            const uint32_t nv = (uint32_t)__popc(lo) + (uint32_t)__popc(hi);
            const uint32_t l0 = i0 - t0, l1 = i1 - t0;
            vix[slot] = l0 | (l1 << 6) | ((uint32_t)p0 << 12) | ((uint32_t)p1 << 13) | ((uint32_t)(nv > 32u) << 14);
            if constexpr (!F16) {
                const float *vp = reinterpret_cast<const float *>(vals_base) + t0;
                vb0[slot] = (uint32_t)lane < nv ? __float_as_uint(__ldg(vp + lane)) : 0u;
                vb1[slot] = nv > 32u && (uint32_t)lane + 32u < nv ? __float_as_uint(__ldg(vp + 32 + lane)) : 0u;
            } else {
                const unsigned short *vp = reinterpret_cast<const unsigned short *>(vals_base) + t0;
                vb0[slot] = (uint32_t)lane < nv ? (uint32_t)__ldg(vp + lane) : 0u;
                vb1[slot] = nv > 32u && (uint32_t)lane + 32u < nv ? (uint32_t)__ldg(vp + 32 + lane) : 0u;
            }
        } else if constexpr (PF256 == 2) {  // values with an L2 evict-first policy (measurement variant)
            if constexpr (!F16) {
                const uint32_t *vp = reinterpret_cast<const uint32_t *>(p.vals);
                uint32_t x0 = 0u, x1 = 0u;
                if (p0) ldg_nc(x0, vp + i0, pol_stream);
                if (p1) ldg_nc(x1, vp + i1, pol_stream);
                vb0[slot] = x0;
                vb1[slot] = x1;
            } else {
                const unsigned short *vp = reinterpret_cast<const unsigned short *>(p.vals);
                vb0[slot] = p0 ? (uint32_t)__ldg(vp + i0) : 0u;
                vb1[slot] = p1 ? (uint32_t)__ldg(vp + i1) : 0u;
            }
        } else if constexpr (PF256 == 1) {
            if constexpr (!F16) {
                const uint32_t *vp = reinterpret_cast<const uint32_t *>(p.vals);
                vb0[slot] = p0 ? ldg_pf256_u32(vp + i0) : 0u;
                vb1[slot] = p1 ? ldg_pf256_u32(vp + i1) : 0u;
            } else {
                const unsigned short *vp = reinterpret_cast<const unsigned short *>(p.vals);
                vb0[slot] = p0 ? ldg_pf256_u16(vp + i0) : 0u;
                vb1[slot] = p1 ? ldg_pf256_u16(vp + i1) : 0u;
            }
        } else if constexpr (VST > 0) {  // values staged in shared memory (or from L2 on overflow)
            const uint32_t vlo = sm.vlo[(j / CH) & 1];
            if constexpr (!F16) {
                const uint32_t *vs = reinterpret_cast<const uint32_t *>(sm.vals[(j / CH) & 1]);
                const uint32_t *vp = reinterpret_cast<const uint32_t *>(p.vals);
                vb0[slot] = p0 ? (vlo != 0xFFFFFFFFu ? vs[i0 - vlo] : __ldg(vp + i0)) : 0u;
                vb1[slot] = p1 ? (vlo != 0xFFFFFFFFu ? vs[i1 - vlo] : __ldg(vp + i1)) : 0u;
            } else {
                const unsigned short *vs = reinterpret_cast<const unsigned short *>(sm.vals[(j / CH) & 1]);
                const unsigned short *vp = reinterpret_cast<const unsigned short *>(p.vals);
                vb0[slot] = p0 ? (uint32_t)(vlo != 0xFFFFFFFFu ? vs[i0 - vlo] : __ldg(vp + i0)) : 0u;
                vb1[slot] = p1 ? (uint32_t)(vlo != 0xFFFFFFFFu ? vs[i1 - vlo] : __ldg(vp + i1)) : 0u;
            }
        } else if constexpr (!F16) {
            const float *vp = reinterpret_cast<const float *>(vals_base);
            vb0[slot] = p0 ? __float_as_uint(__ldg(vp + i0)) : 0u;
            vb1[slot] = p1 ? __float_as_uint(__ldg(vp + i1)) : 0u;
            if constexpr (NH == 2) {  // word 1 (rows 8-15): its values follow all of word 0's
                const uint64_t m1 = c.mask[cs * 2 + 1];
                const uint32_t lo = (uint32_t)m1, hi = (uint32_t)(m1 >> 32);
                const uint32_t r = (hw ? hi : lo) >> p0w;
                const uint32_t j0 = t0 + (uint32_t)__popcll(mask) + (uint32_t)__popc(lo & m_lo) +
                                    (uint32_t)__popc(hi & m_hi);
                const uint32_t j1 = j0 + (uint32_t)__popc(r & ((1u << DK) - 1u));
                vc0[slot & SM1] = (r & 1u) ? __float_as_uint(__ldg(vp + j0)) : 0u;
                vc1[slot & SM1] = ((r >> DK) & 1u) ? __float_as_uint(__ldg(vp + j1)) : 0u;
            }
        } else {
            // keep the two halves apart until the MMA: packing here would stall on the loads
            const unsigned short *vp = reinterpret_cast<const unsigned short *>(vals_base);
            vb0[slot] = p0 ? (uint32_t)__ldg(vp + i0) : 0u;
            vb1[slot] = p1 ? (uint32_t)__ldg(vp + i1) : 0u;
            if constexpr (NH == 2) {
                const uint64_t m1 = c.mask[cs * 2 + 1];
                const uint32_t lo = (uint32_t)m1, hi = (uint32_t)(m1 >> 32);
                const uint32_t r = (hw ? hi : lo) >> p0w;
                const uint32_t j0 = t0 + (uint32_t)__popcll(mask) + (uint32_t)__popc(lo & m_lo) +
                                    (uint32_t)__popc(hi & m_hi);
                const uint32_t j1 = j0 + (uint32_t)__popc(r & ((1u << DK) - 1u));
                vc0[slot & SM1] = (r & 1u) ? (uint32_t)__ldg(vp + j0) : 0u;
                vc1[slot & SM1] = ((r >> DK) & 1u) ? (uint32_t)__ldg(vp + j1) : 0u;
            }
        }
    };

    // ---- lane 0: two gather4 of block j's B rows into stage s
    // ---- HYB, all lanes: block j's 8 B rows into stage s by 16-byte cp.async, in the TMA's
    // layout (gather x / y rows, row stride RS, FP16 y rows 16 bytes in); padding lanes are
    // zero-filled (src-size 0); one noinc arrival per lane on the stage barrier
    auto issue_ldgsts = [&](uint32_t j, int s) {
        const auto &c = sm.ch[(j / CH) % NCB];
        const uint32_t cs = j & (CH - 1u);
        constexpr int CPR = FW * CF::ES / 16;  // 16-byte chunks per gathered row
        const char *Bb = reinterpret_cast<const char *>(p.B) + f0 * CF::ES;
        const int64_t rstride = p.N * CF::ES;
        const uint32_t st = smem_u32(sm.stage[s]);
#pragma unroll
        for (int q0 = 0; q0 < 8 * CPR; q0 += 32) {
            const int q = q0 + lane;
            if (8 * CPR % 32 == 0 || q < 8 * CPR) {
                const int r = q / CPR, cc = q % CPR;
                const uint32_t row = c.a2b[cs * 8 + r];
                const int gsel = F16 ? (r & 1) : (r >> 2);
                const int slot = F16 ? (r >> 1) : (r & 3);
                const uint32_t shift = (LDSM && gsel) ? 16u : 0u;
                const uint32_t dst = st + (uint32_t)(gsel * GC::GRP + slot * GC::RS) + shift + (uint32_t)(cc * 16);
                const bool pad = row == kPadLane;
                const char *src = pad ? Bb : Bb + (int64_t)row * rstride + cc * 16;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(pad ? 0 : 16)
                             : "memory");
            }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&sm.bar[s * BSTR])) : "memory");
    };
    auto issue_tma = [&](uint32_t j, int s) {
        if constexpr (HYB) {
            if (s == 1) {
                issue_ldgsts(j, s);
                return;
            }
        }
        // EL 0: lane 0 issues; 1: an elect.sync lane issues (the body is its branch); 2: every
        // lane computes the operands (broadcast LDS), only the arrive and the two TMA issues are
        // predicated on the elected lane, so no divergent branch remains
        const bool leader = EL == 0 ? lane == 0 : EL == 1 ? elect_one() : true;
        if (leader) {
            const auto &c = sm.ch[(j / CH) % NCB];
            const uint32_t cs = j & (CH - 1u);
            // padding lanes hold 0xFFFFFFFF on the device (row -1): the TMA zero-fills them
            const uint4 ca = *reinterpret_cast<const uint4 *>(&c.a2b[cs * 8]);
            const uint4 cb = *reinterpret_cast<const uint4 *>(&c.a2b[cs * 8 + 4]);
            // hot columns (R22): the block's tag picks its L2 policy (HT = false: untagged plan,
            // instantiated without this code -- it sits on the TMA issue path of every block)
            const uint64_t pol = HT && (ca.x >> kHotShift) > (uint32_t)p.hot_lim ? pol_stream : pol_keep;
            const uint32_t x0 = HT ? ca.x & p.id_mask : ca.x;
            const int32_t r0 = (int32_t)x0, r1 = (int32_t)ca.y, r2 = (int32_t)ca.z, r3 = (int32_t)ca.w;
            const int32_t r4 = (int32_t)cb.x, r5 = (int32_t)cb.y, r6 = (int32_t)cb.z, r7 = (int32_t)cb.w;
            const uint32_t bar = smem_u32(&sm.bar[s * BSTR]);
            const uint32_t st = smem_u32(sm.stage[s]);
            // no proxy fence: the stage's previous generic reads fed this warp's mma.sync,
            // which cannot issue before every lane's LDS has returned
            const bool one = EL == 2 ? elect_one() : true;
            if (one) mbar_arrive_expect_tx(bar, 8u * RS);
            // derived here, not held across the loop (registers are the occupancy limit)
            const CUtensorMap *tmap = &maps.m[NM > 1 ? slice : 0];
            const int32_t tcol = NM > 1 ? 0 : slice * (B3 ? 3 * FW / 2 : FW);  // in map elements
            const int32_t tcol_y = LDSM ? tcol - 8 : tcol;
            if (one) {
                if constexpr (!F16) {
                    tma_gather4(st, tmap, tcol, r0, r1, r2, r3, bar, pol);
                    tma_gather4(st + GC::GRP, tmap, tcol, r4, r5, r6, r7, bar, pol);
                } else {
                    tma_gather4(st, tmap, tcol, r0, r2, r4, r6, bar, pol);
                    tma_gather4(st + GC::GRP, tmap, tcol_y, r1, r3, r5, r7, bar, pol);
                }
            }
        }
    };

    float acc[MT][4];
    float acc1[NH == 2 ? MT : 1][4];  // window rows 8-15 (WH = 16)
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
    if constexpr (NH == 2) {
#pragma unroll
        for (int m = 0; m < MT; ++m) acc1[m][0] = acc1[m][1] = acc1[m][2] = acc1[m][3] = 0.f;
    }

    // ---- consumer: wait for stage s, load the gathered-row fragments, tensor-core MMA
    auto consume = [&](uint32_t i, int s, int slot) {
        mbar_wait_t<WT>(smem_u32(&sm.bar[s * BSTR]), (i / STAGES) & 1u);
        if constexpr (PF256 == 3) {  // pick this lane's two values out of the warp's value run
            const uint32_t ix = vix[slot], l0 = ix & 63u, l1 = (ix >> 6) & 63u;
            uint32_t a0 = __shfl_sync(0xffffffffu, vb0[slot], (int)(l0 & 31u));
            uint32_t a1 = __shfl_sync(0xffffffffu, vb0[slot], (int)(l1 & 31u));
            if (ix & (1u << 14)) {  // warp-uniform: the block holds more than 32 values
                const uint32_t c0 = __shfl_sync(0xffffffffu, vb1[slot], (int)(l0 & 31u));
                const uint32_t c1 = __shfl_sync(0xffffffffu, vb1[slot], (int)(l1 & 31u));
                a0 = l0 >= 32u ? c0 : a0;
                a1 = l1 >= 32u ? c1 : a1;
            }
            vb0[slot] = (ix & (1u << 12)) ? a0 : 0u;
            vb1[slot] = (ix & (1u << 13)) ? a1 : 0u;
        }
        const uint8_t *st = sm.stage[s];
        const uint8_t *ra = st + frag_off;
        const uint8_t *rb = st + GC::GRP + frag_off;
        if constexpr (L64) {
#pragma unroll
            for (int j = 0; j < FW / 32; ++j) {
#pragma unroll
                for (int tau = 0; tau < 2; ++tau) {
                    uint2 xa = *reinterpret_cast<const uint2 *>(ra + 128 * j + 16 * tau);
                    uint2 ya = *reinterpret_cast<const uint2 *>(rb + 128 * j + 16 * tau);
                    if constexpr (RND) {
                        xa = make_uint2(tf32_rna_bits(xa.x), tf32_rna_bits(xa.y));
                        ya = make_uint2(tf32_rna_bits(ya.x), tf32_rna_bits(ya.y));
                    }
                    mma_tf32(acc[2 * j + tau], xa.x, xa.y, ya.x, ya.y, vb0[slot], vb1[slot]);
                    if constexpr (NH == 2) {
                        mma_tf32(acc1[2 * j + tau], xa.x, xa.y, ya.x, ya.y, vc0[slot & SM1], vc1[slot & SM1]);
                    }
                }
            }
        } else if constexpr (B3) {
            // rows t (k = t, gather x) and t + 4 (gather y); per 8-feature group j: LDS.128 of the
            // high halves + LDS.64 of the bytes 15..8; one PRMT per element rebuilds the TF32
            // operand (byte 0 is don't-care: the tensor core reads bits 31..13 only)
            const uint8_t *xa = st + t * GC::RS, *ya = st + GC::GRP + t * GC::RS;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const uint4 hx = *reinterpret_cast<const uint4 *>(xa + 128 * j + 16 * g);
                const uint2 lx = *reinterpret_cast<const uint2 *>(xa + 2 * FW + 64 * j + 8 * g);
                const uint4 hy = *reinterpret_cast<const uint4 *>(ya + 128 * j + 16 * g);
                const uint2 ly = *reinterpret_cast<const uint2 *>(ya + 2 * FW + 64 * j + 8 * g);
                const uint32_t hxs[4] = {hx.x, hx.y, hx.z, hx.w}, hys[4] = {hy.x, hy.y, hy.z, hy.w};
                uint32_t xv[8], yv[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const uint32_t sel = (e & 1) ? (0x3202u | ((4u + (e & 3)) << 4)) : (0x1000u | ((4u + (e & 3)) << 4));
                    xv[e] = __byte_perm(hxs[e >> 1], e < 4 ? lx.x : lx.y, sel);
                    yv[e] = __byte_perm(hys[e >> 1], e < 4 ? ly.x : ly.y, sel);
                }
                if constexpr (K8) {  // FW = 64: one m16n8k8 per tile (k = t from x, t + 4 from y)
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        mma_tf32(acc[4 * j + q], xv[2 * q], xv[2 * q + 1], yv[2 * q], yv[2 * q + 1], vb0[slot], vb1[slot]);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) mma_tf32_k4(acc[4 * j + q], xv[2 * q], xv[2 * q + 1], vb0[slot]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) mma_tf32_k4(acc[4 * j + q], yv[2 * q], yv[2 * q + 1], vb1[slot]);
                }
            }
        } else if constexpr (LDSM) {
            // lane L addresses row k = L & 7 of matrix L >> 3 (8 features); k even in gather x,
            // k odd in gather y (+16 B: its column window starts 8 features early)
            const int k = lane & 7, mx = lane >> 3;
            const uint32_t row = smem_u32(st) + ((k & 1) ? GC::GRP + 16u : 0u) + (uint32_t)(k >> 1) * GC::RS;
            const uint32_t bv = vb0[slot] | (vb1[slot] << 16);
            const uint32_t bw = NH == 2 ? (vc0[slot & SM1] | (vc1[slot & SM1] << 16)) : 0u;
            if constexpr (FW >= 32) {
#pragma unroll
                for (int q = 0; q < FW / 32; ++q) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4_trans(a0, a1, a2, a3, row + (uint32_t)(mx * 16 + q * 64));
                    mma_f16(acc[2 * q], a0, a1, bv);
                    mma_f16(acc[2 * q + 1], a2, a3, bv);
                    if constexpr (NH == 2) {
                        mma_f16(acc1[2 * q], a0, a1, bw);
                        mma_f16(acc1[2 * q + 1], a2, a3, bw);
                    }
                }
            } else {
                uint32_t a0, a1;
                ldsm_x2_trans(a0, a1, row + (uint32_t)((mx & 1) * 16));
                mma_f16(acc[0], a0, a1, bv);
                if constexpr (NH == 2) mma_f16(acc1[0], a0, a1, bw);
            }
        } else if constexpr (!F16 && CF::VW == 4) {
            // two k=4 halves of the 8x8 tile: rows t (k = 0..3) and t+4 (k = 4..7); each
            // LDS.128 of one row feeds the A operands of two m16 tiles directly.  All k = 0..3
            // MMAs go first so dependent accumulations sit NV*2 instructions apart.
            uint4 x[NV], y[NV];
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                x[j] = *reinterpret_cast<const uint4 *>(ra + 8 * CF::VB * j);
                y[j] = *reinterpret_cast<const uint4 *>(rb + 8 * CF::VB * j);
                if constexpr (RND) {  // rho(B) in registers (low-reuse plans skip the pre-round pass)
                    x[j] = make_uint4(tf32_rna_bits(x[j].x), tf32_rna_bits(x[j].y), tf32_rna_bits(x[j].z),
                                      tf32_rna_bits(x[j].w));
                    y[j] = make_uint4(tf32_rna_bits(y[j].x), tf32_rna_bits(y[j].y), tf32_rna_bits(y[j].z),
                                      tf32_rna_bits(y[j].w));
                }
            }
            if constexpr (K8) {  // one m16n8k8 per m16 tile: (x.x, x.y) k = t, (y.x, y.y) k = t + 4
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    mma_tf32(acc[2 * j], x[j].x, x[j].y, y[j].x, y[j].y, vb0[slot], vb1[slot]);
                    mma_tf32(acc[2 * j + 1], x[j].z, x[j].w, y[j].z, y[j].w, vb0[slot], vb1[slot]);
                }
                if constexpr (NH == 2) {
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        mma_tf32(acc1[2 * j], x[j].x, x[j].y, y[j].x, y[j].y, vc0[slot & SM1], vc1[slot & SM1]);
                        mma_tf32(acc1[2 * j + 1], x[j].z, x[j].w, y[j].z, y[j].w, vc0[slot & SM1], vc1[slot & SM1]);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    mma_tf32_k4(acc[2 * j], x[j].x, x[j].y, vb0[slot]);
                    mma_tf32_k4(acc[2 * j + 1], x[j].z, x[j].w, vb0[slot]);
                }
                if constexpr (NH == 2) {
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        mma_tf32_k4(acc1[2 * j], x[j].x, x[j].y, vc0[slot & SM1]);
                        mma_tf32_k4(acc1[2 * j + 1], x[j].z, x[j].w, vc0[slot & SM1]);
                    }
                }
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    mma_tf32_k4(acc[2 * j], y[j].x, y[j].y, vb1[slot]);
                    mma_tf32_k4(acc[2 * j + 1], y[j].z, y[j].w, vb1[slot]);
                }
                if constexpr (NH == 2) {
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        mma_tf32_k4(acc1[2 * j], y[j].x, y[j].y, vc1[slot & SM1]);
                        mma_tf32_k4(acc1[2 * j + 1], y[j].z, y[j].w, vc1[slot & SM1]);
                    }
                }
            }
        } else {
            Frag<FW, F16> fr;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                fr.x[j] = *reinterpret_cast<const V *>(ra + 8 * CF::VB * j);
                fr.y[j] = *reinterpret_cast<const V *>(rb + 8 * CF::VB * j);
            }
            if constexpr (RND) round_frag<FW, F16>(fr);
            if constexpr (F16) {
                fr.b0 = vb0[slot] | (vb1[slot] << 16);
                fr.b1 = 0u;
            } else {
                fr.b0 = vb0[slot];
                fr.b1 = vb1[slot];
            }
            mma_block<FW, F16>(acc, fr);
            if constexpr (NH == 2) {
                if constexpr (F16) {
                    fr.b0 = vc0[slot & SM1] | (vc1[slot & SM1] << 16);
                } else {
                    fr.b0 = vc0[slot & SM1];
                    fr.b1 = vc1[slot & SM1];
                }
                mma_block<FW, F16>(acc1, fr);
            }
        }
    };

    // a = the accumulator half of window rows lr0 .. lr0 + 7 (WH = 16: acc, then acc1 at lr0 + 8)
    auto store_rows = [&](float *base, int64_t ld, int64_t lr0, bool remap, const uint32_t *rmap, auto &a) {
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int64_t lr = lr0 + 2 * t + s2;
            if (!remap || lr < p.rows) {
                const int64_t orow = remap ? (rmap ? (int64_t)__ldg(rmap + lr) : lr) : lr;
                if constexpr (L64) {  // tile 2j + tau: features 32j + 2 slot(g, tau) + {0, 1}
                    float *d = base + orow * ld + 2 * l64_slot;
#pragma unroll
                    for (int j = 0; j < FW / 32; ++j)
#pragma unroll
                        for (int tau = 0; tau < 2; ++tau)
                            st_cs(d + 32 * j + 4 * tau, a[2 * j + tau][s2], a[2 * j + tau][2 + s2]);
                    continue;
                }
                if constexpr (LDSM) {  // tile mt: features 16mt + g (c0/c1) and 16mt + 8 + g (c2/c3)
                    float *d = base + orow * ld + g;
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        st_cs1(d + 16 * mt, a[mt][s2]);
                        st_cs1(d + 16 * mt + 8, a[mt][2 + s2]);
                    }
                    continue;
                }
                float *dst = base + orow * ld + VW * g;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    float *d = dst + 8 * VW * j;
                    if constexpr (VW == 2) {
                        st_cs(d, a[j][s2], a[j][2 + s2]);
                    } else {
#pragma unroll
                        for (int q = 0; q < VW / 4; ++q) {
                            const int m0 = (VW / 2) * j + 2 * q;
                            st_cs(d + 4 * q, a[m0][s2], a[m0][2 + s2], a[m0 + 1][s2], a[m0 + 1][2 + s2]);
                        }
                    }
                }
            }
        }
    };
    auto store_window = [&](uint32_t wi) {
        const int64_t lr0 = (int64_t)(w0 + wi) * WH;
        if (p.ndst == 0) {
            store_rows(p.C + f0, p.N, lr0, true, p.row_map, acc);
            if constexpr (NH == 2) store_rows(p.C + f0, p.N, lr0 + 8, true, p.row_map, acc1);
        } else {  // fused all-gather: the rows go straight to every rank's C (original order)
#pragma unroll 1
            for (int d = 0; d < p.ndst; ++d) {
                store_rows(p.dst[d] + f0, p.N, lr0, true, p.orig_map, acc);
                if constexpr (NH == 2) store_rows(p.dst[d] + f0, p.N, lr0 + 8, true, p.orig_map, acc1);
            }
        }
#pragma unroll
        for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
        if constexpr (NH == 2) {
#pragma unroll
            for (int m = 0; m < MT; ++m) acc1[m][0] = acc1[m][1] = acc1[m][2] = acc1[m][3] = 0.f;
        }
    };
    // split-window fixup: add one segment's partial tile (rows 0-7 of it) into accumulator a
    auto add_tile = [&](const float *src, auto &a) {
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            if constexpr (L64) {
                const float *row = src + (2 * t + s2) * FW + 2 * l64_slot;
#pragma unroll
                for (int j = 0; j < FW / 32; ++j)
#pragma unroll
                    for (int tau = 0; tau < 2; ++tau) {
                        const float2 v = __ldcg(reinterpret_cast<const float2 *>(row + 32 * j + 4 * tau));
                        a[2 * j + tau][s2] += v.x;
                        a[2 * j + tau][2 + s2] += v.y;
                    }
                continue;
            }
            if constexpr (LDSM) {
                const float *row = src + (2 * t + s2) * FW + g;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    a[mt][s2] += __ldcg(row + 16 * mt);
                    a[mt][2 + s2] += __ldcg(row + 16 * mt + 8);
                }
                continue;
            }
            const float *row = src + (2 * t + s2) * FW + VW * g;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
#pragma unroll
                for (int e = 0; e < VW; e += 2) {
                    const int m = (VW / 2) * j + (e >> 1);
                    const float2 v = __ldcg(reinterpret_cast<const float2 *>(row + 8 * VW * j + e));
                    a[m][s2] += v.x;
                    a[m][2 + s2] += v.y;
                }
            }
        }
    };
    // wend = absolute block index where the current window ends; 0xFFFFFFFF once no whole
    // window is left (split units, or after the last one): one compare per block
    uint32_t wi = 0;
    uint32_t wend = __shfl_sync(0xffffffffu, my_rwo, 1);
    if (split || nw == 0) wend = 0xFFFFFFFFu;
    auto after_block = [&](uint32_t jnext) {
        while (wend == jnext) {
            store_window(wi);
            ++wi;
            const uint32_t e = __shfl_sync(0xffffffffu, my_rwo, (int)(wi < nw ? wi + 1 : nw));
            wend = wi < nw ? e : 0xFFFFFFFFu;
        }
    };

    // Prologue: chunk 0 (wait) and chunk 1 in flight; values of block 0; TMA of block 0.
    // With value staging: chunks 0 and 1 landed, chunk 2 in flight, values of chunks 0 (waited)
    // and 1 in flight.
    issue_chunk(0);
    if constexpr (VST > 0) issue_chunk(CH);
    cp_async_wait_all();
    __syncwarp();
    issue_chunk(VST > 0 ? 2 * CH : CH);
    if constexpr (VST > 0) {
        issue_vals(0);
        issue_vals(1);
        if (nblk > 0) mbar_wait(smem_u32(&sm.vbar[0]), 0);
    }
    after_block(b0);
    if (nblk > 0) value_load(0u, 0);
    if (!DYN && VD == 2 && nblk > 1) value_load(1u, 1);
    if (nblk > 0) issue_tma(0, 0);
    if constexpr (DYN) {
        // Deep ring with a run-time stage index (measurement variant): block step j issues the
        // TMA and loads the values of jt = j + L (L = STAGES - 1), then consumes block j.  The
        // unroll is the 4-slot value ring only (the stage rotates at run time), so the loop
        // body stays as small as the default one.  Chunk c + 1 is staged once jt has entered
        // chunk c: every reader of chunk c - 1's buffer (TMA issue, value decode of blocks
        // < c * CH) has then run.
        constexpr int L = STAGES - 1;
#pragma unroll
        for (int d = 1; d < L; ++d)
            if ((uint32_t)d < nblk) {
                issue_tma((uint32_t)d, d);
                value_load((uint32_t)d, d);
            }
        int s_c = 0, s_t = L;
        auto stepD = [&](uint32_t j, int u, bool checked) {
            const uint32_t jt = j + L;
            if ((jt & (CH - 1u)) == 0) {
                cp_async_wait_all();
                __syncwarp();
                issue_chunk(jt + CH);
            }
            if (!checked || jt < nblk) {
                issue_tma(jt, s_t);
                value_load(jt, (u + L) & (VR - 1));
            }
            consume(j, s_c, u & (VR - 1));
            after_block(b0 + j + 1);
            s_c = s_c == STAGES - 1 ? 0 : s_c + 1;
            s_t = s_t == STAGES - 1 ? 0 : s_t + 1;
        };
        const uint32_t nmainD = nblk >= (uint32_t)L ? ((nblk - L) / VR) * VR : 0u;
        uint32_t j = 0;
        for (; j < nmainD; j += VR) {
#pragma unroll
            for (int u = 0; u < VR; ++u) stepD(j + (uint32_t)u, u, false);
        }
        for (; j < nblk; j += VR) {
#pragma unroll
            for (int u = 0; u < VR; ++u)
                if (j + (uint32_t)u < nblk) stepD(j + (uint32_t)u, u, true);
        }
    } else if constexpr (STAGES > 2) {
        // Deeper TMA ring (STAGES - 1 blocks of lookahead; pays where a stage is small, e.g.
        // FP16): block step j issues the TMA of jt = j + L and the values of jn = j + 1.
        // Chunk c + 1 is staged when jn enters chunk c (chunk c - 1's buffer is then free)
        // and waited for when jt enters it.
        static_assert(VD == 1 && STAGES <= 4, "multi-stage ring: one value slot ahead, <= 4 stages");
        constexpr int L = STAGES - 1;
        constexpr int UN = STAGES == 3 ? 6 : 4;  // unroll: a multiple of VR and of STAGES
#pragma unroll
        for (int d = 1; d < L; ++d)
            if ((uint32_t)d < nblk) issue_tma((uint32_t)d, d);
        auto stepS = [&](uint32_t j, int u, bool checked) {
            const uint32_t jn = j + 1, jt = j + L;
            if ((jt & (CH - 1u)) == 0) {
                cp_async_wait_all();
                __syncwarp();
            }
            if ((jn & (CH - 1u)) == 0) issue_chunk(jn + CH);
            if (!checked || jt < nblk) issue_tma(jt, (u + L) % STAGES);
            if (!checked || jn < nblk) value_load(jn, (u + 1) & (VR - 1));
            consume(j, u % STAGES, u & (VR - 1));
            after_block(b0 + j + 1);
        };
        const uint32_t nmainS = nblk >= (uint32_t)L ? ((nblk - L) / UN) * UN : 0u;
        uint32_t j = 0;
        for (; j < nmainS; j += UN) {
#pragma unroll
            for (int u = 0; u < UN; ++u) stepS(j + (uint32_t)u, u, false);
        }
        for (; j < nblk; j += UN) {
#pragma unroll
            for (int u = 0; u < UN; ++u)
                if (j + (uint32_t)u < nblk) stepS(j + (uint32_t)u, u, true);
        }
    } else {
    // Block step j: TMA for j+1, values for j+1 (at a chunk boundary first wait for that
    // chunk and prefetch the one after), then the decode-free MMA of block j.
    auto step = [&](uint32_t j, int u, bool checked) {
        const uint32_t jn = j + 1;
        if constexpr (VD == 1) {
            if ((jn & (CH - 1u)) == 0) {  // chunk (jn / CH) must have landed
                cp_async_wait_all();
                __syncwarp();
                if constexpr (VST > 0) {  // c = jn / CH: metadata c + 2, values c + 1, wait values c
                    const uint32_t c = jn / CH;
                    issue_chunk(jn + 2 * CH);
                    issue_vals(c + 1);
                    if (jn < nblk) mbar_wait(smem_u32(&sm.vbar[c & 1]), (c >> 1) & 1u);
                } else {
                    issue_chunk(jn + CH);
                }
            }
            if (!checked || jn < nblk) {
                issue_tma(jn, (u + 1) & 1);
                value_load(jn, (u + 1) & (VR - 1));
            }
        } else {
            // the TMA of jn reads its row ids before chunk jv + CH may overwrite jn's buffer
            const uint32_t jv = j + 2;
            if (!checked || jn < nblk) issue_tma(jn, (u + 1) & 1);
            if ((jv & (CH - 1u)) == 0) {
                cp_async_wait_all();
                __syncwarp();
                issue_chunk(jv + CH);
            }
            if (!checked || jv < nblk) value_load(jv, (u + 2) & (VR - 1));
        }
        consume(j, u & 1, u & (VR - 1));
        after_block(b0 + j + 1);
    };
    const uint32_t nmain = nblk >= (uint32_t)VD ? ((nblk - VD) / VR) * VR : 0u;
    uint32_t j = 0;
    for (; j < nmain; j += VR) {
#pragma unroll
        for (int u = 0; u < VR; ++u) step(j + (uint32_t)u, u, false);
    }
    for (; j < nblk; j += VR) {
#pragma unroll
        for (int u = 0; u < VR; ++u)
            if (j + (uint32_t)u < nblk) step(j + (uint32_t)u, u, true);
    }
    }
    cp_async_wait_all();

    if (split) {
        const uint32_t sid = ub.x, seg = ub.y, nseg = ub.z, slot = ub.w;
        float *tile = p.ws + ((int64_t)slot * p.nslices + slice) * (WH * FW);
        store_rows(tile, FW, 0, false, nullptr, acc);
        if constexpr (NH == 2) store_rows(tile, FW, 8, false, nullptr, acc1);
        __threadfence();
        __syncwarp();
        uint32_t prev = 0;
        if (lane == 0) prev = atomicAdd(p.counters + (int64_t)sid * p.nslices + slice, 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == nseg - 1) {
            __threadfence();
            const float *first = p.ws + ((int64_t)(slot - seg) * p.nslices + slice) * (WH * FW);
#pragma unroll
            for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
            if constexpr (NH == 2) {
#pragma unroll
                for (int m = 0; m < MT; ++m) acc1[m][0] = acc1[m][1] = acc1[m][2] = acc1[m][3] = 0.f;
            }
            for (uint32_t k = 0; k < nseg; ++k) {
                const float *src = first + (int64_t)k * p.nslices * (WH * FW);
                if constexpr (NH == 2) add_tile(src + 8 * FW, acc1);
                add_tile(src, acc);
            }
            store_window(0);
            if (lane == 0) p.counters[(int64_t)sid * p.nslices + slice] = 0u;
        }
    }
}

// B -> TF32 (RNA) once per execute; each B row is then gathered by many windows.
__global__ void round_b_tf32_kernel(const float4 *__restrict__ in, float4 *__restrict__ out, int64_t n4)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
        float4 v = __ldcs(in + e);
        uint32_t a, b, c, d;
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(a) : "f"(v.x));
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(b) : "f"(v.y));
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(c) : "f"(v.z));
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(d) : "f"(v.w));
        out[e] = make_float4(__uint_as_float(a), __uint_as_float(b), __uint_as_float(c), __uint_as_float(d));
    }
}

#ifdef ACCSPMM_VARIANTS
// rho(B) into the 3-byte TF32 image B3 (G4Cfg): output row r, feature slice s (FW wide) =
// FW high halves (bits 31..16) then FW bytes (bits 15..8) of rho(B[src][s*FW + f]), src = perm[r]
// with permuted columns (R18), else r.  rho(b) has bits 12..0 zero, so the image is lossless.
// One warp per row, one float4 (4 features) per lane step.
__global__ void pack_b3_kernel(const float4 *__restrict__ in, uint8_t *__restrict__ out, const uint32_t *__restrict__ perm,
                               int64_t K, int64_t N, int FW)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t n4 = N / 4;
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < K; r += warps) {
        const float4 *src = in + (perm ? (int64_t)__ldg(perm + r) : r) * n4;
        uint8_t *dst = out + r * 3 * N;
        for (int64_t i = lane; i < n4; i += 32) {
            const float4 v = __ldcs(src + i);
            const uint32_t x0 = tf32_rna_bits(__float_as_uint(v.x)), x1 = tf32_rna_bits(__float_as_uint(v.y));
            const uint32_t x2 = tf32_rna_bits(__float_as_uint(v.z)), x3 = tf32_rna_bits(__float_as_uint(v.w));
            const int64_t f = 4 * i, sl = f / FW, fl = f - sl * FW;
            uint8_t *o = dst + sl * 3 * FW;
            *reinterpret_cast<uint2 *>(o + 2 * fl) = make_uint2(__byte_perm(x0, x1, 0x7632), __byte_perm(x2, x3, 0x7632));
            *reinterpret_cast<uint32_t *>(o + 2 * FW + fl) = __byte_perm(__byte_perm(x0, x1, 0x0051), __byte_perm(x2, x3, 0x0051), 0x5410);
        }
    }
}

#endif  // ACCSPMM_VARIANTS

// ------------------------------------------------------------------ launch

#ifdef ACCSPMM_VARIANTS
template <int FW, bool F16, int WARPS, bool RND = false>
accspmm_status launch_cfg(const KParams &kp, int64_t n_units, cudaStream_t stream)
{
    auto kern = spmm_bittcf_kernel<FW, F16, WARPS, RND>;
    const int64_t groups = (n_units + WARPS - 1) / WARPS;
    const int64_t grid = groups * kp.nslices;
    if (grid > 0x7FFFFFFFll) return fail(ACCSPMM_ERR_UNSUPPORTED, "grid too large");
    kern<<<(unsigned)grid, WARPS * 32, 0, stream>>>(kp);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("spmm launch: ") + cudaGetErrorString(e));
    return ACCSPMM_OK;
}
#endif

// NM = 1: one tensor map (the full-width map when several slices exist); NM = kMaxSliceMaps:
// one map per slice (tensor_map decides; only the default configurations instantiate it)
template <int FW, bool F16, int WARPS, int STAGES, bool RND = false, int MINB = 1, int NM = 1, bool LDSM = false,
          bool K8 = false, int VD = 1, int PF256 = 0, int VST = 0, bool HYB = false, int CX = (VST ? 4 : 0),
          bool B3 = false, bool DEC64 = false, int EL = 1, bool HT = true, bool PIN = false, bool DYN = false,
          int BS = 1, int WT = 0, int WH = 8, bool L64 = false, int PAD = 0>
accspmm_status launch_g4(const KParams &kp, const G4Maps *map, int64_t n_units, cudaStream_t stream)
{
    using SM = G4Smem<FW, F16, STAGES, VST, CX, B3, BS, WH / 8, PAD>;
    const size_t smem = sizeof(SM) * WARPS;
    auto kern = spmm_bittcf_g4_kernel<FW, F16, WARPS, STAGES, RND, MINB, NM, LDSM, K8, VD, PF256, VST, HYB, CX, B3, DEC64, EL, HT, PIN, DYN, BS, WT, WH, L64, PAD>;
    static int configured_device = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_device != dev) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
        // the whole unified L1/shared array as shared memory: occupancy is smem-limited
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
        configured_device = dev;
    }
    const int64_t groups = (n_units + WARPS - 1) / WARPS;
    const int64_t grid = groups * kp.nslices;
    if (grid > 0x7FFFFFFFll) return fail(ACCSPMM_ERR_UNSUPPORTED, "grid too large");
    kern<<<(unsigned)grid, WARPS * 32, smem, stream>>>(kp, *reinterpret_cast<const G4MapsT<NM> *>(map));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("spmm launch: ") + cudaGetErrorString(e));
    return ACCSPMM_OK;
}

// TMA tensor maps of B (2D: K rows x width columns, box = BOXE x 1 for gather4), cached in
// the plan; one per feature slice when the slices fit G4Maps (see G4Maps)
// b3: B is the 3-byte TF32 image (3N bytes per row, slices of 3FW bytes, u16 map elements)
accspmm_status tensor_map(const DevicePlan &d, const KParams &kp, int FW, bool multi, bool b3, const G4Maps **out,
                          bool l64 = false)
{
    const void *B = kp.B;
    const int64_t N = kp.N;
    const int nm = multi ? map_count(kp) : 1;
    const int pv = knobs().l2promo;
    const uint64_t key[4] = {(uint64_t)(uintptr_t)B, (uint64_t)N, (uint64_t)FW,
                             (uint64_t)(d.precision + 1) | ((uint64_t)nm << 8) | ((uint64_t)pv << 16) |
                                 ((uint64_t)b3 << 24) | ((uint64_t)l64 << 25)};
    G4Maps *maps = reinterpret_cast<G4Maps *>(d.tmap);
    static_assert(sizeof(G4Maps) <= sizeof(d.tmap), "tensor-map cache too small");
    if (!(key[0] == d.tmap_key[0] && key[1] == d.tmap_key[1] && key[2] == d.tmap_key[2] && key[3] == d.tmap_key[3])) {
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        if (!encode) {
            cudaDriverEntryPointQueryResult q;
            void *fn = nullptr;
            cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
            if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
                return fail(ACCSPMM_ERR_CUDA, "cuTensorMapEncodeTiled entry point not available");
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        }
        const bool f16 = d.precision == ACCSPMM_FP16;
        const cuuint64_t es = f16 ? 2 : 4;
        // L2 sector promotion of the gathered rows (Knobs::l2promo 0..3 = none/64/128/256 B
        // for A/B measurements in the variants build; default 256 B)
        const CUtensorMapL2promotion promo = pv == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                            : pv == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                            : pv == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                      : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
        for (int m = 0; m < nm; ++m) {
            // B3: a row is 3N bytes = 3N/2 u16 elements, slice m starts at byte 3*FW*m
            const cuuint64_t slice_e = b3 ? 3 * FW / 2 : FW, row_e = b3 ? 3 * N / 2 : N;
            cuuint64_t dims[2] = {(cuuint64_t)(nm > 1 ? slice_e : row_e), (cuuint64_t)d.K};
            cuuint64_t strides[1] = {(cuuint64_t)(b3 ? 3 * N : N * es)};
            // G4Cfg::BOXE: the slice plus 32 bytes
            // (L64: the slice plus 16 bytes)
            cuuint32_t box[2] = {(cuuint32_t)(b3 ? (3 * FW + 32) / 2 : FW + (f16 ? 16 : l64 ? 4 : 8)), 1u};
            cuuint32_t estr[2] = {1u, 1u};
            void *base = const_cast<char *>(reinterpret_cast<const char *>(B)) + (size_t)m * FW * (b3 ? 3 : es);
            CUresult r = encode(&maps->m[m], (f16 || b3) ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
                                base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS)
                return fail(ACCSPMM_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
        }
        for (int k = 0; k < 4; ++k) d.tmap_key[k] = key[k];
    }
    *out = maps;
    return ACCSPMM_OK;
}

// Minimum resident warps per SM for __launch_bounds__ (caps registers per thread): the
// kernel is latency-bound, so occupancy pays until the register cap starts to serialise
// the gather/decode pipeline.  Measured on the Reddit-shaped and stencil matrices
// (DESIGN.md §7): FW 128 20 (TF32 is then smem-bound; FP16 spills above); FW 64/32 24;
// FW 16 32.
template <int FW, bool F16>
constexpr int tuned_min_warps()
{
    return FW == 128 ? 20 : FW == 16 ? 32 : 24;
}

template <int FW, bool F16>
accspmm_status launch_fw(const KParams &kp, const DevicePlan &d, const void *B, int64_t n_units, cudaStream_t stream,
                         bool rnd, bool b3)
{
    // Default (measured): TMA gather4, one warp x 2 stages per CTA (the warp's
    // shared-memory addresses are then CTA constants, so the TMA operands need few uniform-
    // register moves), tuned launch bounds, one tensor map per feature slice when N > FW.
    // FP16 takes its A fragments by ldmatrix.trans.
    constexpr int MW = tuned_min_warps<FW, F16>();
    // all-gather and hot-column plans (lane-0 tags): the default kernel (or a B3 variant)
    const int kcfg = (kp.ndst > 0 || (kp.hot_lim != 255 && !is_b3_variant(knobs().kcfg))) ? -1 : knobs().kcfg;
    const G4Maps *map = nullptr;
    // per-slice maps only for the kernels instantiated with them (variants 20/46: one map)
    const bool multi = map_count(kp) > 1 && kcfg != 20 && kcfg != 46;
    static const G4Maps no_maps = {};  // no TC blocks (e.g. K = 0): no TMA is ever issued
    if (kcfg < 0 || kcfg >= 20) {
        // L64 layout (kcfg 87): TF32 rows FW + 4 elements apart
        const bool l64 = !F16 && FW >= 32 && !rnd && kcfg == 87 && d.wh == 8;
        accspmm_status st = d.NB > 0 ? tensor_map(d, kp, FW, multi, b3, &map, l64) : (map = &no_maps, ACCSPMM_OK);
        if (st != ACCSPMM_OK) return st;
    }
    constexpr int NM = kMaxSliceMaps;
    constexpr bool LD = F16;       // FP16: ldmatrix.trans fragments (measured -10.5%)
    constexpr bool K8 = FW <= 64;  // TF32: one m16n8k8 per tile at FW <= 64 (-6% at N = 64)
#ifdef ACCSPMM_VARIANTS
    if constexpr (!F16 && FW >= 64) {
        // TF32 with a pre-rounded B gathered from its 3-byte image (G4Cfg B3; measured, not
        // taken: DESIGN.md §7 -- the kernel is issue/latency-bound, the 24% fewer gathered
        // bytes do not offset the 32 PRMT per block that rebuild the operands)
        if (b3 && kcfg == 58) {  // B3 with values two blocks ahead (4-slot value ring)
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, false, K8, 2, 0, 0, false, 0, true>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, false, K8, 2, 0, 0, false, 0, true>(kp, map, n_units, stream);
        }
        if (b3 && kcfg == 60) {  // B3, 3-stage TMA ring (2 blocks of lookahead), 18 warps per SM
            if (multi) return launch_g4<FW, F16, 1, 3, false, 18, NM, false, K8, 1, 0, 0, false, 0, true>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 3, false, 18, 1, false, K8, 1, 0, 0, false, 0, true>(kp, map, n_units, stream);
        }
        if (b3 && kcfg == 61) {  // B3, 4-stage TMA ring (3 blocks of lookahead), 14 warps per SM
            if (multi) return launch_g4<FW, F16, 1, 4, false, 14, NM, false, K8, 1, 0, 0, false, 0, true>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 4, false, 14, 1, false, K8, 1, 0, 0, false, 0, true>(kp, map, n_units, stream);
        }
        if (b3 && kcfg == 59) {  // B3 with 24 resident warps per SM (register cap 85)
            if (multi) return launch_g4<FW, F16, 1, 2, false, 24, NM, false, K8, 1, 0, 0, false, 0, true>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, 24, 1, false, K8, 1, 0, 0, false, 0, true>(kp, map, n_units, stream);
        }
        if (b3) {
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, false, K8, 1, 0, 0, false, 0, true>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, false, K8, 1, 0, 0, false, 0, true>(kp, map, n_units, stream);
        }
    }
#endif
    if (b3) return fail(ACCSPMM_ERR_INTERNAL, "B3 layout: variants build, TF32, 64/128-feature slices only");
    if (d.wh == 16) {
        // 16-row windows (reading R20) on this kernel: every gathered row feeds two accumulator
        // halves, so the register cap admits fewer resident warps
        constexpr int MW16 = FW == 128 ? 16 : FW == 64 ? 20 : 24;
        if constexpr (!F16) {
            if (rnd) {
                if (multi) return launch_g4<FW, F16, 1, 2, true, MW16, NM, false, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 0, 16>(kp, map, n_units, stream);
                return launch_g4<FW, F16, 1, 2, true, MW16, 1, false, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 0, 16>(kp, map, n_units, stream);
            }
        }
        if (multi) return launch_g4<FW, F16, 1, 2, false, MW16, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 0, 16>(kp, map, n_units, stream);
        return launch_g4<FW, F16, 1, 2, false, MW16, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 0, 16>(kp, map, n_units, stream);
    }
#ifdef ACCSPMM_VARIANTS
    // Measured-and-rejected alternatives, selectable by ACCSPMM_KCFG in the variants build only
    // (libaccspmm_variants.so): 20 = 2 warps per CTA without a launch-bounds minimum (the
    // round-1 kernel), 46 = 2 warps per CTA with tuned bounds, 47 = FP16 fragments by LDS.128 +
    // PRMT, 48 = the other TF32 k4/k8 choice, 49 = values two blocks ahead, 50/51 = 3/4-stage
    // TMA ring, 52 = value loads with an L2 256-byte prefetch, 10-12 = register-direct gather.
    if (kcfg >= 0 && kcfg < 20) {
        if constexpr (!F16) {
            if (rnd) return launch_cfg<FW, F16, 2, true>(kp, n_units, stream);
        }
        switch (kcfg) {
        case 10: return launch_cfg<FW, F16, 4>(kp, n_units, stream);
        case 12: return launch_cfg<FW, F16, 8>(kp, n_units, stream);
        default: return launch_cfg<FW, F16, 2>(kp, n_units, stream);
        }
    }
    if constexpr (!F16) {
        if (rnd) {  // B not pre-rounded: rho(B) applied in registers
            if (kcfg == 20) return launch_g4<FW, F16, 2, 2, true, 1>(kp, map, n_units, stream);
            if (kcfg == 52) {
                if (multi) return launch_g4<FW, F16, 1, 2, true, MW, NM, false, K8, 1, 1>(kp, map, n_units, stream);
                return launch_g4<FW, F16, 1, 2, true, MW, 1, false, K8, 1, 1>(kp, map, n_units, stream);
            }
        }
    }
    if (!rnd) {
        switch (kcfg) {
        case 20: return launch_g4<FW, F16, 2, 2, false, 1>(kp, map, n_units, stream);
        case 46: return launch_g4<FW, F16, 2, 2, false, MW / 2>(kp, map, n_units, stream);
        case 48:
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, !K8>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, !K8>(kp, map, n_units, stream);
        case 52:
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 1>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 1>(kp, map, n_units, stream);
        case 56:  // hybrid gather: odd blocks by cp.async, even blocks by TMA
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, true>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, true>(kp, map, n_units, stream);
        case 54:  // chunk values staged by bulk copy (256 per chunk buffer)
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 256>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 256>(kp, map, n_units, stream);
        case 55:  // chunk values staged by bulk copy (512 per chunk buffer)
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 512>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 512>(kp, map, n_units, stream);
        case 63:  // default kernel with the TMA issued under lane == 0 instead of elect.sync
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 0>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 0>(kp, map, n_units, stream);
        case 64:  // TMA operands computed by every lane, only the arrive + issues elected (EL 2)
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 2, false>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 2, false>(kp, map, n_units, stream);
        case 68:  // 4 more resident warps per SM than the tuned launch bound (register cap lower)
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW + 4, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW + 4, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
        case 69:  // 4 fewer resident warps per SM than the tuned launch bound
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW - 4, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW - 4, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
        case 66:  // lane constants and the value base pinned in registers (no rematerialisation)
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, true>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, true>(kp, map, n_units, stream);
        case 65:  // values two blocks ahead (4-slot value ring) on the current default (untagged)
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 2, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 2, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
        case 70:  // deep ring: 3 stages, TMA and values 2 blocks ahead, run-time stage index
            if (multi) return launch_g4<FW, F16, 1, 3, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, true>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 3, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, true>(kp, map, n_units, stream);
        case 73:  // values by one coalesced warp load per block + shuffles (PF256 3)
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 3, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 3, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
        case 77:  // default kernel, one 16-byte slot per stage barrier
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 2>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 2>(kp, map, n_units, stream);
        case 78:  // default kernel, one 128-byte line per stage barrier
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 16>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 16>(kp, map, n_units, stream);
        case 79:  // default kernel, stage wait by try_wait without a suspend hint
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 1>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 1>(kp, map, n_units, stream);
        case 80:  // default kernel, stage wait by test_wait spin
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 2>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 2>(kp, map, n_units, stream);
        case 85:  // default kernel, stage barriers packed at the head of the warp's area
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 0, 0>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 0, 0>(kp, map, n_units, stream);
        case 87:  // TF32 FW >= 32: m16n8k8 fed by two LDS.64 per tile (L64 layout, no register moves)
            if constexpr (!F16 && FW >= 32) {
                if (d.wh != 8) break;
                if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 0, 8, true>(kp, map, n_units, stream);
                return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 0, 8, true>(kp, map, n_units, stream);
            }
            break;
        case 93:  // default ring + 128 B of padding per CTA
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 0, 8, false, 128>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false, false, false, 1, 0, 8, false, 128>(kp, map, n_units, stream);
        case 62:  // default kernel with the 64-bit shift decode (tile_rank) instead of the 32-bit one
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, true>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, true>(kp, map, n_units, stream);
        case 57:  // default kernel with the value-staging chunk stride (layout A/B)
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 4>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 4>(kp, map, n_units, stream);
        case 53:  // value loads with an L2 evict-first policy
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 2>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 2>(kp, map, n_units, stream);
        case 50:
            if (multi) return launch_g4<FW, F16, 1, 3, false, MW, NM, LD, K8>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 3, false, MW, 1, LD, K8>(kp, map, n_units, stream);
        case 51:
            if (multi) return launch_g4<FW, F16, 1, 4, false, MW, NM, LD, K8>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 4, false, MW, 1, LD, K8>(kp, map, n_units, stream);
        case 49:
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 2>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 2>(kp, map, n_units, stream);
        case 47:
            if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, false, MW>(kp, map, n_units, stream);
        default: break;
        }
    }
#endif
    // the default kernel, with hot-column tag handling only for tagged plans (R22)
    const bool ht = kp.hot_lim != 255;
    if constexpr (!F16) {
        if (rnd) {  // B not pre-rounded: rho(B) applied in registers
            if (ht) {
                if (multi) return launch_g4<FW, F16, 1, 2, true, MW, NM, false, K8, 1, 0, 0, false, 0, false, false, 1, true>(kp, map, n_units, stream);
                return launch_g4<FW, F16, 1, 2, true, MW, 1, false, K8, 1, 0, 0, false, 0, false, false, 1, true>(kp, map, n_units, stream);
            }
            if (multi) return launch_g4<FW, F16, 1, 2, true, MW, NM, false, K8, 1, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
            return launch_g4<FW, F16, 1, 2, true, MW, 1, false, K8, 1, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
        }
    }
    if (ht) {
        if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, true>(kp, map, n_units, stream);
        return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, true>(kp, map, n_units, stream);
    }
    if (multi) return launch_g4<FW, F16, 1, 2, false, MW, NM, LD, K8, 1, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
    return launch_g4<FW, F16, 1, 2, false, MW, 1, LD, K8, 1, 0, 0, false, 0, false, false, 1, false>(kp, map, n_units, stream);
}

}  // namespace

int pick_fw(int64_t N)
{
    const int f = knobs().fw;
    if ((f == 16 || f == 32 || f == 64 || f == 128) && N % f == 0) return f;
    return N % 128 == 0 ? 128 : N % 64 == 0 ? 64 : N % 32 == 0 ? 32 : 16;
}

accspmm_status launch_round_b(const float *B, float *Br, int64_t n, void *stream)
{
    const int64_t n4 = n / 4;
    int64_t grid = (n4 + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    if (grid < 1) grid = 1;
    round_b_tf32_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const float4 *>(B),
                                                                        reinterpret_cast<float4 *>(Br), n4);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("round launch: ") + cudaGetErrorString(e));
    return ACCSPMM_OK;
}

accspmm_status launch_pack_b3(const float *B, void *out, const uint32_t *perm, int64_t K, int64_t N, int FW, void *stream)
{
#ifndef ACCSPMM_VARIANTS
    (void)B; (void)out; (void)perm; (void)N; (void)FW; (void)stream;
    return fail(ACCSPMM_ERR_INTERNAL, "B3 layout: variants build only");
#else
    if (K == 0) return ACCSPMM_OK;
    int64_t grid = (K + 7) / 8;
    if (grid > 148 * 16) grid = 148 * 16;
    pack_b3_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const float4 *>(B),
                                                                   reinterpret_cast<uint8_t *>(out), perm, K, N, FW);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("pack_b3 launch: ") + cudaGetErrorString(e));
    return ACCSPMM_OK;
#endif
}

accspmm_status launch_spmm(const DevicePlan &d, const void *B, const void *zrow, int64_t N, float *C, float *ws,
                           uint32_t *counters, void *stream, bool round_b, float *const *dst, int ndst, bool b3)
{
    if (d.rows == 0) return ACCSPMM_OK;
    const int FW = pick_fw(N);
    KParams kp;
    kp.rwo = d.rwo;
    kp.tco = d.tco;
    kp.a2b = d.a2b;
    kp.bits = d.bits;
    kp.vals = d.vals;
    kp.units = reinterpret_cast<const uint4 *>(d.units);
    kp.row_map = d.row_map;
    kp.B = B;
    kp.zrow = zrow;
    kp.C = C;
    kp.ws = ws;
    kp.counters = counters;
    kp.N = N;
    kp.rows = d.rows;
    kp.n_units = d.n_units;
    kp.nslices = (int32_t)(N / FW);
    kp.Krows = (int32_t)d.K;
    kp.ndst = ndst;
    // hot columns (R22): with B larger than kHotL2Bytes the hot set is the 2^hot_lim hottest
    // columns whose rows fit kHotBytes; otherwise every block keeps evict_last (hot_lim = 31)
    kp.hot_lim = 255;
    kp.id_mask = d.hot ? kHotIdMask : 0xFFFFFFFFu;
    if (d.hot) {
        const int64_t es = d.precision == ACCSPMM_FP16 ? 2 : 4;
        const int64_t row = N * es, bbytes = d.K * row;
        int lim = 31;
        if (bbytes > knobs().hot_l2_bytes) {
            const int64_t h = std::max<int64_t>(1, knobs().hot_bytes / row);
            lim = 63 - __builtin_clzll((unsigned long long)h);  // 2^lim <= h
        }
        kp.hot_lim = lim;
    }
    // slice-major grid when N spans several slices: one 128-wide slice of B at a time is the L2
    // working set (N = 512: -13%, N = 256: -3%; Knobs::slice_major = 0 restores slice-fastest)
    kp.slice_major = knobs().slice_major != 0 && kp.nslices > 1;
    kp.orig_map = d.orig_map ? d.orig_map : d.row_map;
    for (int k = 0; k < kMaxGatherDst; ++k) kp.dst[k] = k < ndst ? dst[k] : nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    const bool f16 = d.precision == ACCSPMM_FP16;
    const bool r = round_b;
    switch (FW) {
    case 128: return f16 ? launch_fw<128, true>(kp, d, B, d.n_units, s, r, b3) : launch_fw<128, false>(kp, d, B, d.n_units, s, r, b3);
    case 64: return f16 ? launch_fw<64, true>(kp, d, B, d.n_units, s, r, b3) : launch_fw<64, false>(kp, d, B, d.n_units, s, r, b3);
    case 32: return f16 ? launch_fw<32, true>(kp, d, B, d.n_units, s, r, b3) : launch_fw<32, false>(kp, d, B, d.n_units, s, r, b3);
    default: return f16 ? launch_fw<16, true>(kp, d, B, d.n_units, s, r, b3) : launch_fw<16, false>(kp, d, B, d.n_units, s, r, b3);
    }
}

}  // namespace accspmm
