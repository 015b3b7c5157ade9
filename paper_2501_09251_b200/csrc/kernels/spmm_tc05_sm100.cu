// Acc-SpMM on the 5th-generation tensor cores (tcgen05 + TMEM), sm_100a -- SURVEY NEXT-1.
//
// What it computes is the same product as spmm_sm100.cu: every TC block of a RowWindow
// is decoded from its occupancy bitmap with the popcount rule of P:273 and
// multiplied against the gathered rows of B with the operands swapped: the
// gathered B rows are the left operand (M = 128 features x K = 8 gathered rows), the decoded
// sparse tile the right operand (K = 8 x N = window rows).  TF32 inputs, FP32 accumulation
// (P:308).  Windows may be taller than the paper's 8 rows (reading R20: wh = 16 / 32 rows,
// wh x 8 tiles), which cuts the dominant gathered-row bytes (Reddit-shaped, reordered:
// sum_w |U_w| -14% at 16 rows, -28% at 32) at the price of wh/8 times the MMA work per
// gathered row -- affordable only on tcgen05.
//
// Data path of one TC block (one CTA = 4 warps = one work unit x one 128-feature slice):
//   L2 --(TMA tile::gather4, 2 per block, leader thread)--> shared stage (8 rows x 512 B)
//      --(LDS.32: thread = feature, 8 rows)--> registers --(tcgen05.st 32x32b.x8)--> TMEM A[s]
//   bitmap + values --(decode)--> shared B tile (K-major, no swizzle: core matrices of
//      8 window rows x 16 B)
//   leader: tcgen05.mma.cta_group::1.kind::tf32 D[tmem] (+)= A[tmem] . B[smem desc];
//           tcgen05.commit -> "empty" mbarrier of the stage; at a window's end -> "acc" mbarrier
//   window end: tcgen05.ld 32x32b (thread = feature, one column per window row) -> st.global
// The gathered rows are MN-major (features contiguous), which UMMA reads from shared memory
// only in the 128-byte-swizzled layout (one TMA request per 4 rows x 32 features: 8 per
// block instead of 2); the transposition through registers into TMEM (the
// A-from-TMEM "TS" form) keeps the gather at 2 TMA requests per block.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../internal.hpp"

namespace accspmm {
namespace {

constexpr int kFW = 128;    // features per CTA slice = UMMA M
constexpr int kCH = 16;     // TC blocks per staged A-stream chunk
constexpr int kThreads = 128;
constexpr int kStageBytes = 8 * kFW * 4;  // 8 gathered rows x 128 features x 4 B

struct TcParams {
    const uint32_t *__restrict__ rwo;
    const uint32_t *__restrict__ tco;
    const uint32_t *__restrict__ a2b;
    const uint64_t *__restrict__ bits;
    const float *__restrict__ vals;
    const uint4 *__restrict__ units;
    const uint32_t *__restrict__ row_map;
    float *__restrict__ C;
    float *__restrict__ ws;
    uint32_t *__restrict__ counters;
    int64_t N;
    int64_t rows;
    int64_t n_units;
    int32_t nslices;
    int32_t wh;         // rows per window of the plan (<= HT)
    int32_t nw;         // occupancy words per block = wh / 8
    int32_t slice_major;
};


// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
// Waits on an mbarrier phase.  WM = 0: try_wait with a suspend-time hint (the thread may
// sleep until the phase completes); 1: test_wait spin (never sleeps); 2: try_wait without hint.
template <int WM>
__device__ __forceinline__ void mbar_wait_m(uint32_t bar, uint32_t phase)
{
    if constexpr (WM == 1) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "WAIT_%=:\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar), "r"(phase)
            : "memory");
    } else if constexpr (WM == 2) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar), "r"(phase)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
            "@P1 bra DONE_%=;\n\t"
            "bra WAIT_%=;\n\t"
            "DONE_%=:\n\t}\n" ::"r"(bar), "r"(phase), "r"(0x989680)
            : "memory");
    }
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

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap *map, int32_t col, int32_t r0, int32_t r1,
                                            int32_t r2, int32_t r3, uint32_t bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// TMEM <- registers: 32 lanes (one per thread of the warp) x 8 consecutive 32-bit columns
__device__ __forceinline__ void tmem_st_x8(uint32_t taddr, const uint32_t (&v)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// registers <- TMEM: 32 lanes x 16 consecutive columns
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&v)[16], int off)
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr + (uint32_t)off)
        : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]: M = 128, N = HT, K = 8, TF32 in, FP32 accumulate
__device__ __forceinline__ void umma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                 : "memory");
}

// Shared-memory matrix descriptor of the B tile: K-major, no swizzle (canonical
// ((8,n),2):((1,SBO),LBO) in 16-byte units): core matrix = 8 window rows x 16 B (4 TF32 of K),
// LBO = 128 B between the two K halves, SBO = 256 B between 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t btile_desc(uint32_t saddr)
{
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32) |
           (1ull << 46);
}

__device__ __forceinline__ uint32_t tf32_rna_bits(uint32_t x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(__uint_as_float(x)));
    return r;
}

// ------------------------------------------------------------------ the kernel
//
// Warp roles (160 threads): warps 0-3 = transposers (thread = feature of the 128-feature
// slice: TMEM lane quarter = warp; lanes < HT/4 also decode one tile row each), warp 4 lane 0 =
// producer: A-stream chunk and value bulk copies, B-row gathers (TMA), MMAs.  They synchronise only through mbarriers:
//   chunk_full[2]  bulk copies of a chunk's SparseAToB / TCLocalBit / TCOffset (tx bytes)
//   vals_full[2]   bulk copy of the chunk's value range (or an overflow flag: values from L2)
//   full_t[ST]     TMA gather of a block's 8 B rows (tx bytes)
//   ready[SA]      4 transposer warps: A[sa] in TMEM and their rows of the decoded tile B[sa]
//   empty[SA]      tcgen05.commit: the MMA that read A[sa] / B[sa] has completed
//   acc_full[ND]   tcgen05.commit after a window's (segment's) last MMA
//   acc_free[ND]   4 transposer warps: accumulator read back, D may be overwritten
// A chunk buffer is refilled only after the ready[] of the chunk's last block (every reader
// is done with it); a gather stage only after the ready[] of the block it held.

#ifdef ACCSPMM_VARIANTS
// phase-cycle trace of the first kTraceCtas CTAs (variants build, kcfg 68): [cta][slot]
constexpr int kTraceCtas = 64, kTraceSlots = 16;
__device__ unsigned long long g_tc05_trace[kTraceCtas * kTraceSlots];
#endif

template <int HT, int ST, int SA, int ND>
struct TcLayout {
    static constexpr int NWMAX = HT / 8;
    static constexpr int VCAP = 512;                                  // staged values per chunk
    static constexpr int STAGE = 0;                                   // ST x 4096
    static constexpr int BTILE = STAGE + ST * kStageBytes;            // SA x HT x 8 x 4
    static constexpr int A2B = BTILE + SA * HT * 32;                  // 2 x CH x 8 u32
    static constexpr int BITS = A2B + 2 * kCH * 8 * 4;                // 2 x (CH x NWMAX + 2) u64
    static constexpr int BITS_BUF = kCH * NWMAX + 2;
    static constexpr int TCO = BITS + 2 * BITS_BUF * 8;               // 2 x (CH + 8) u32
    static constexpr int TCO_BUF = kCH + 8;
    static constexpr int VALS = (TCO + 2 * TCO_BUF * 4 + 15) / 16 * 16;  // 2 x (VCAP + 8) f32
    static constexpr int VALS_BUF = VCAP + 8;
    static constexpr int BAR = VALS + 2 * VALS_BUF * 4;               // mbarriers
    static constexpr int NBAR = 2 + 2 + ST + 2 * SA + 2 * ND;
    static constexpr int MISC = BAR + NBAR * 8;                       // tmem base, chunk offsets
    static constexpr int BYTES = MISC + 64;
    static constexpr int TMEM_NEED = SA * 8 + ND * HT;
    static constexpr int TMEM_COLS = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128 : 256;
};

__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// CP = commit period: one tcgen05.commit frees CP consecutive A / B stages (CP divides SA)
template <int HT, int ST, int SA, int ND, bool RND, int WM = 0, int CP = 1, int REP = 1, bool TR = false>
__global__ void __launch_bounds__(kThreads + 32, 6)
    spmm_tc05_kernel(const TcParams p, const __grid_constant__ CUtensorMap tmap)
{
    // TR: accumulate clock64 cycles per phase into g_tc05_trace (one transposer lane, the producer)
    const bool trace_on = TR && blockIdx.x < 64;
    unsigned long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tr_t = TR ? clock64() : 0;
    auto mark = [&](int slot) {
        if constexpr (TR) {
            const long long t = clock64();
            tr[slot] += (unsigned long long)(t - tr_t);
            tr_t = t;
        }
    };
    static_assert(SA % CP == 0, "commit period must divide the stage count");
    auto mbar_wait = [](uint32_t bar, uint32_t phase) { mbar_wait_m<WM>(bar, phase); };
    using L = TcLayout<HT, ST, SA, ND>;
    constexpr int NWMAX = L::NWMAX;
    // instruction descriptor: D F32 (bit 4), A/B TF32 (bits 7, 10), K-major A and B,
    // N >> 3 at bit 17, M >> 4 at bit 24 (M = 128)
    constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(HT >> 3) << 17) | (8u << 24);
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *stage = smem + L::STAGE;
    float *btile = reinterpret_cast<float *>(smem + L::BTILE);
    uint32_t *ch_a2b = reinterpret_cast<uint32_t *>(smem + L::A2B);
    uint64_t *ch_bits = reinterpret_cast<uint64_t *>(smem + L::BITS);
    uint32_t *ch_tco = reinterpret_cast<uint32_t *>(smem + L::TCO);
    float *ch_vals = reinterpret_cast<float *>(smem + L::VALS);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::BAR);
    // misc[0] = TMEM base; misc[4 + buf] = word shift of ch_bits; misc[6 + buf] = entry shift of
    // ch_tco; misc[8 + buf] = first value index staged (0xFFFFFFFF: overflow, values from L2);
    // misc[12] = split-window arrival count
    uint32_t *misc = reinterpret_cast<uint32_t *>(smem + L::MISC);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned ngrp = (unsigned)p.n_units;
    const int slice = p.slice_major ? (int)(blockIdx.x / ngrp) : (int)(blockIdx.x % (unsigned)p.nslices);
    const int64_t u = p.slice_major ? (int64_t)(blockIdx.x % ngrp) : (int64_t)(blockIdx.x / (unsigned)p.nslices);
    const int64_t f0 = (int64_t)slice * kFW;

    const uint4 ua = __ldg(p.units + 2 * u);
    const uint4 ub = __ldg(p.units + 2 * u + 1);
    const uint32_t w0 = ua.x, nwin = ua.y, b0 = ua.z, b1 = ua.w;
    const bool split = ub.x != kNoSplit;
    const uint32_t nblk = b1 - b0;
    const uint32_t my_rwo = (uint32_t)lane <= nwin ? __ldg(p.rwo + w0 + lane) : 0u;

    const uint32_t bar0 = smem_u32(bars);
    auto chunk_full = [&](int b) { return bar0 + 8u * (uint32_t)b; };
    auto vals_full = [&](int b) { return bar0 + 8u * (uint32_t)(2 + b); };
    auto full_t = [&](int s) { return bar0 + 8u * (uint32_t)(4 + s); };
    auto ready = [&](int s) { return bar0 + 8u * (uint32_t)(4 + ST + s); };
    // empty barrier of the stage group holding block j (groups of CP stages)
    auto empty = [&](uint32_t j) { return bar0 + 8u * (uint32_t)(4 + ST + SA + (int)((j / CP) % (SA / CP))); };
    auto acc_full = [&](int d) { return bar0 + 8u * (uint32_t)(4 + ST + 2 * SA + d); };
    auto acc_free = [&](int d) { return bar0 + 8u * (uint32_t)(4 + ST + 2 * SA + ND + d); };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(misc)),
                     "r"((uint32_t)L::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (tid == kThreads) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
        for (int b = 0; b < 2; ++b) {
            mbar_init(chunk_full(b), 1);
            mbar_init(vals_full(b), 1);
        }
        for (int s = 0; s < ST; ++s) mbar_init(full_t(s), 1);
        for (int s = 0; s < SA; ++s) {
            mbar_init(ready(s), 4);
            mbar_init(bar0 + 8u * (uint32_t)(4 + ST + SA + s), 1);
        }
        for (int d = 0; d < ND; ++d) {
            mbar_init(acc_full(d), 1);
            mbar_init(acc_free(d), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc[0];

    // window bookkeeping (identical in every warp): wend = absolute end block of window wi
    auto first_wend = [&]() { return split ? b1 : __shfl_sync(0xffffffffu, my_rwo, 1); };

    if (warp == 4) {
        // ============================== producer (lane 0): chunk / value copies, gathers, MMAs
        const uint64_t pol_keep = policy_evict_last();
        // chunk c (blocks [c*CH, +CH)) into buffer c & 1: 16-byte-aligned supersets of the
        // arrays by bulk copy (the allocations carry the padding)
        auto issue_chunk = [&](uint32_t c) {
            const uint32_t i = c * kCH;
            if (i >= nblk) return;
            const int buf = c & 1;
            const uint32_t b = b0 + i;
            const uint32_t cnt = min((uint32_t)kCH, nblk - i);
            const uint32_t w_lo = (b * (uint32_t)p.nw) & ~1u, w_hi = ((b + cnt) * (uint32_t)p.nw + 1u) & ~1u;
            const uint32_t t_lo = b & ~3u, t_hi = (b + cnt + 1u + 3u) & ~3u;
            misc[4 + buf] = b * (uint32_t)p.nw - w_lo;
            misc[6 + buf] = b - t_lo;
            const uint32_t bytes = cnt * 32u + (w_hi - w_lo) * 8u + (t_hi - t_lo) * 4u;
            mbar_arrive_expect_tx(chunk_full(buf), bytes);
            bulk_g2s(smem_u32(ch_a2b + buf * kCH * 8), p.a2b + (size_t)b * 8, cnt * 32u, chunk_full(buf));
            bulk_g2s(smem_u32(ch_bits + buf * L::BITS_BUF), p.bits + w_lo, (w_hi - w_lo) * 8u, chunk_full(buf));
            bulk_g2s(smem_u32(ch_tco + buf * L::TCO_BUF), p.tco + t_lo, (t_hi - t_lo) * 4u, chunk_full(buf));
        };
        // values of chunk c (after its TCOffset landed): [tco[first], tco[last + 1]) superset
        auto issue_vals = [&](uint32_t c) {
            const uint32_t i = c * kCH;
            if (i >= nblk) return;
            const int buf = c & 1;
            const uint32_t cnt = min((uint32_t)kCH, nblk - i);
            const uint32_t *tc = ch_tco + buf * L::TCO_BUF + misc[6 + buf];
            const uint32_t v_lo = tc[0] & ~3u, v_hi = (tc[cnt] + 3u) & ~3u;
            if (v_hi - v_lo <= (uint32_t)L::VCAP) {
                misc[8 + buf] = v_lo;
                mbar_arrive_expect_tx(vals_full(buf), (v_hi - v_lo) * 4u);
                if (v_hi > v_lo)
                    bulk_g2s(smem_u32(ch_vals + buf * L::VALS_BUF), p.vals + v_lo, (v_hi - v_lo) * 4u, vals_full(buf));
            } else {
                misc[8 + buf] = 0xFFFFFFFFu;  // too many values for the stage: read from L2
                mbar_arrive(vals_full(buf));
            }
        };
        auto issue_tma = [&](uint32_t j, int s) {
            const int buf = (j / kCH) & 1;
            const uint32_t cs = j & (kCH - 1u);
            const uint4 ca = *reinterpret_cast<const uint4 *>(&ch_a2b[(buf * kCH + cs) * 8]);
            const uint4 cb = *reinterpret_cast<const uint4 *>(&ch_a2b[(buf * kCH + cs) * 8 + 4]);
            const uint32_t bar = full_t(s);
            const uint32_t dst = smem_u32(stage + s * kStageBytes);
            mbar_arrive_expect_tx(bar, (uint32_t)kStageBytes);
            const int32_t col = (int32_t)f0;
            tma_gather4(dst, &tmap, col, (int32_t)ca.x, (int32_t)ca.y, (int32_t)ca.z, (int32_t)ca.w, bar, pol_keep);
            tma_gather4(dst + kStageBytes / 2, &tmap, col, (int32_t)cb.x, (int32_t)cb.y, (int32_t)cb.z,
                        (int32_t)cb.w, bar, pol_keep);
        };
        if (nblk == 0 || lane != 0) return;
        // window of the block cursor (the transposers zero-write the empty ones)
        uint32_t wi = 0, wend = split ? b1 : __ldg(p.rwo + w0 + 1);
        auto advance = [&](uint32_t cursor) {
            while (!split && wi < nwin && wend == cursor) {
                ++wi;
                wend = wi < nwin ? __ldg(p.rwo + w0 + wi + 1) : 0xFFFFFFFFu;
            }
        };
        advance(b0);
        issue_chunk(0);
        issue_chunk(1);
        mbar_wait(chunk_full(0), 0);
        issue_vals(0);
        for (int s = 0; s < ST; ++s)
            if ((uint32_t)s < nblk) issue_tma((uint32_t)s, s);
        bool first = true;
        uint32_t accn = 0;  // accumulations started (window or segment)
        for (uint32_t j = 0; j < nblk; ++j) {
            const int sa = (int)(j % SA);
            const uint32_t cs = j & (kCH - 1u);
            const uint32_t jb = b0 + j;
            const bool last = split ? (j + 1 == nblk) : (jb + 1 == wend);
            {
                mark(7);
                if (first && accn >= (uint32_t)ND)  // D[accn % ND] read back by the transposers?
                    mbar_wait(acc_free(accn % ND), ((accn / ND) - 1u) & 1u);
                mark(0);
                mbar_wait(ready(sa), (j / SA) & 1u);
                mark(1);
                tc_fence_after();
                const int dsel = (int)(accn % ND);
                umma_tf32_ts(tmem + (uint32_t)(SA * 8 + dsel * HT), tmem + (uint32_t)(sa * 8),
                             btile_desc(smem_u32(btile + sa * HT * 8)), IDESC, first ? 0u : 1u);
                // REP > 1 (variants build, timing probe only -- wrong results): the tensor core
                // executes every block's MMA REP times
                for (int rep = 1; rep < REP; ++rep)
                    umma_tf32_ts(tmem + (uint32_t)(SA * 8 + dsel * HT), tmem + (uint32_t)(sa * 8),
                                 btile_desc(smem_u32(btile + sa * HT * 8)), IDESC, 1u);
                if ((j % CP) == CP - 1 || j + 1 == nblk) umma_commit(empty(j));
                if (last) umma_commit(acc_full(dsel));
                mark(2);
                // chunk c fully consumed once the ready[] of its last block is in: refill with c + 2
                if (cs == kCH - 1u) issue_chunk(j / kCH + 2);
                const uint32_t jt = j + ST;  // gather of block jt into the stage block j vacated
                if (jt < nblk) {
                    if ((jt & (kCH - 1u)) == 0) {  // first block of chunk jt/CH: metadata must have landed
                        const uint32_t c = jt / kCH;
                        mbar_wait(chunk_full(c & 1), (c >> 1) & 1u);
                        issue_vals(c);
                    }
                    issue_tma(jt, (int)(j % ST));
                }
                mark(3);
            }
            if (last) {
                ++accn;
                advance(jb + 1);
            }
            first = last;
        }
#ifdef ACCSPMM_VARIANTS
        if (trace_on)
            for (int k = 0; k < 8; ++k) atomicAdd(&g_tc05_trace[blockIdx.x * kTraceSlots + k], tr[k]);
#endif
        return;
    }

    // ===================================================== transposers (warps 0-3)
    const int feat = warp * 32 + lane;                       // feature (TMEM lane) in the slice
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;  // this warp's TMEM lane quarter
    auto store_rows = [&](const uint32_t (&d)[HT], int64_t lr0, float *base, int64_t ld, bool remap) {
#pragma unroll
        for (int n = 0; n < HT; ++n) {
            const int64_t lr = lr0 + n;
            if (n < p.wh) {
                if (remap) {
                    if (lr < p.rows) {
                        const int64_t orow = p.row_map ? (int64_t)__ldg(p.row_map + lr) : lr;
                        __stcs(base + orow * ld + f0 + feat, __uint_as_float(d[n]));
                    }
                } else {
                    __stcg(base + (int64_t)n * ld + feat, __uint_as_float(d[n]));
                }
            }
        }
    };
    // accumulator D[dsel] -> registers, then release it to the MMA issuer
    auto load_acc = [&](uint32_t (&d)[HT], int dsel, uint32_t phase) {
        mbar_wait(acc_full(dsel), phase & 1u);
        tc_fence_after();
        uint32_t t[16];
#pragma unroll
        for (int h = 0; h < HT; h += 16) {
            tmem_ld_x16(tmem + lane_off + (uint32_t)(SA * 8 + dsel * HT), t, h);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q) d[h + q] = t[q];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_free(dsel));
    };
    uint32_t zeros[HT];
#pragma unroll
    for (int q = 0; q < HT; ++q) zeros[q] = 0u;
    auto window_row0 = [&](uint32_t w) { return (int64_t)(w0 + w) * p.wh; };

    uint32_t wi = 0;
    uint32_t wend = first_wend();
    auto skip_empty = [&](uint32_t jb) {  // zero-write windows without blocks at cursor jb
        while (!split && wi < nwin && wend == jb) {
            store_rows(zeros, window_row0(wi), p.C, p.N, true);
            ++wi;
            const uint32_t e = __shfl_sync(0xffffffffu, my_rwo, (int)(wi < nwin ? wi + 1 : nwin));
            wend = wi < nwin ? e : 0xFFFFFFFFu;
        }
    };
    skip_empty(b0);
    uint32_t accn = 0;
    for (uint32_t j = 0; j < nblk; ++j) {
        const int st = (int)(j % ST), sa = (int)(j % SA);
        mark(6);
        if (j >= (uint32_t)SA) mbar_wait(empty(j), ((j / SA) - 1u) & 1u);
        mark(0);
        tc_fence_after();
        mbar_wait(full_t(st), (j / ST) & 1u);
        mark(1);
        {   // gathered rows -> TMEM A[sa]: this thread's feature of the 8 rows
            const float *sp = reinterpret_cast<const float *>(stage + st * kStageBytes);
            uint32_t v[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                v[r] = __float_as_uint(sp[r * kFW + feat]);
                if constexpr (RND) v[r] = tf32_rna_bits(v[r]);
            }
            tmem_st_x8(tmem + lane_off + (uint32_t)(sa * 8), v);
        }
        mark(2);
        {   // decode of this warp's HT/4 tile rows (lane = row): the row's occupancy
            // byte and the rank of its first value -- values ascend by tile position r*8 + lane,
            // so a row's values are one contiguous run -- into B[sa] (K-major core matrices)
            const int buf = (j / kCH) & 1;
            const uint32_t cs = j & (kCH - 1u);
            if (cs == 0) {
                mbar_wait(chunk_full(buf), ((j / kCH) >> 1) & 1u);
                mbar_wait(vals_full(buf), ((j / kCH) >> 1) & 1u);
            }
            constexpr int RPW = HT / 4;  // tile rows per warp
            if (lane < RPW) {
                const int n = warp * RPW + lane;
                float r[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) r[k] = 0.f;
                if (n < p.wh) {
                    const uint64_t *wb = ch_bits + buf * L::BITS_BUF + misc[4 + buf] + cs * (uint32_t)p.nw;
                    const int word = n >> 3, sh = (n & 7) * 8;
                    const uint64_t m = wb[word];
                    const uint32_t byte = (uint32_t)(m >> sh) & 0xFFu;
                    if (byte) {
                        uint32_t idx = ch_tco[buf * L::TCO_BUF + misc[6 + buf] + cs] +
                                       (uint32_t)__popcll(m & ((1ull << sh) - 1ull));
#pragma unroll
                        for (int q = 0; q < NWMAX - 1; ++q)
                            if (q < word) idx += (uint32_t)__popcll(wb[q]);
                        const uint32_t vlo = misc[8 + buf];
                        const float *vsrc =
                            vlo != 0xFFFFFFFFu ? ch_vals + buf * L::VALS_BUF + (idx - vlo) : p.vals + idx;
                        int c = 0;
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            if ((byte >> k) & 1u) r[k] = vsrc[c++];
                    }
                }
                float *bt = btile + sa * HT * 8 + (n >> 3) * 64 + (n & 7) * 4;
                *reinterpret_cast<float4 *>(bt) = make_float4(r[0], r[1], r[2], r[3]);
                *reinterpret_cast<float4 *>(bt + 32) = make_float4(r[4], r[5], r[6], r[7]);
            }
            fence_proxy_async_smem();
        }
        mark(3);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ready(sa));
        mark(4);
        const uint32_t jb = b0 + j;
        const bool last = split ? (j + 1 == nblk) : (jb + 1 == wend);
        if (last && !split) {
            uint32_t d[HT];
            load_acc(d, (int)(accn % ND), accn / ND);
            ++accn;
            store_rows(d, window_row0(wi), p.C, p.N, true);
            ++wi;
            const uint32_t e = __shfl_sync(0xffffffffu, my_rwo, (int)(wi < nwin ? wi + 1 : nwin));
            wend = wi < nwin ? e : 0xFFFFFFFFu;
            skip_empty(jb + 1);
        }
        mark(5);
    }
#ifdef ACCSPMM_VARIANTS
    if (trace_on && warp == 0 && lane == 0)
        for (int k = 0; k < 8; ++k) atomicAdd(&g_tc05_trace[blockIdx.x * kTraceSlots + 8 + k], tr[k]);
#endif

    if (split) {
        // cross-row write-back of a split window (reading R15): partial -> workspace,
        // the last-arriving segment sums the partials in segment order (deterministic)
        const uint32_t sid = ub.x, seg = ub.y, nseg = ub.z, slot = ub.w;
        const int64_t tile_elems = (int64_t)p.wh * kFW;
        float *tile = p.ws + ((int64_t)slot * p.nslices + slice) * tile_elems;
        uint32_t d[HT];
        if (nblk > 0) load_acc(d, 0, 0);
        else {
#pragma unroll
            for (int q = 0; q < HT; ++q) d[q] = 0u;
        }
        store_rows(d, 0, tile, kFW, false);
        __threadfence();
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        if (tid == 0) misc[12] = atomicAdd(p.counters + (int64_t)sid * p.nslices + slice, 1u);
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        if (misc[12] == nseg - 1) {
            __threadfence();
            const float *firstp = p.ws + ((int64_t)(slot - seg) * p.nslices + slice) * tile_elems;
            float acc[HT];
#pragma unroll
            for (int q = 0; q < HT; ++q) acc[q] = 0.f;
            for (uint32_t k = 0; k < nseg; ++k) {
                const float *src = firstp + (int64_t)k * p.nslices * tile_elems;
#pragma unroll
                for (int n = 0; n < HT; ++n)
                    if (n < p.wh) acc[n] += __ldcg(src + (int64_t)n * kFW + feat);
            }
            uint32_t r[HT];
#pragma unroll
            for (int q = 0; q < HT; ++q) r[q] = __float_as_uint(acc[q]);
            store_rows(r, window_row0(0), p.C, p.N, true);
            if (tid == 0) p.counters[(int64_t)sid * p.nslices + slice] = 0u;  // re-arm for the next execute
        }
    }
    // every MMA was waited for (acc_full) before its accumulator was read: free TMEM
    tc_fence_before();
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    tc_fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"((uint32_t)L::TMEM_COLS)
                     : "memory");
}

// ------------------------------------------------------------------ launch

accspmm_status tensor_map_tc05(const DevicePlan &d, const void *B, int64_t N, const CUtensorMap **out)
{
    // key marks this kernel's map (box = exactly one 128-feature slice, no padding columns)
    const uint64_t key[4] = {(uint64_t)(uintptr_t)B, (uint64_t)N, (uint64_t)kFW, 0x7C05ull << 32};
    CUtensorMap *map = reinterpret_cast<CUtensorMap *>(d.tmap);
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
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)d.K};
        cuuint64_t strides[1] = {(cuuint64_t)N * 4};
        cuuint32_t box[2] = {(cuuint32_t)kFW, 1u};
        cuuint32_t estr[2] = {1u, 1u};
        CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(B), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return fail(ACCSPMM_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
        for (int k = 0; k < 4; ++k) d.tmap_key[k] = key[k];
    }
    *out = map;
    return ACCSPMM_OK;
}

template <int HT, int ST, int SA, int ND, bool RND, int WM = 0, int CP = 1, int REP = 1, bool TR = false>
accspmm_status launch_tc(const TcParams &tp, const CUtensorMap *map, cudaStream_t stream)
{
    using L = TcLayout<HT, ST, SA, ND>;
    auto kern = spmm_tc05_kernel<HT, ST, SA, ND, RND, WM, CP, REP, TR>;
    static int configured_device = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_device != dev) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
        if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
        configured_device = dev;
    }
    const int64_t grid = tp.n_units * tp.nslices;
    if (grid > 0x7FFFFFFFll) return fail(ACCSPMM_ERR_UNSUPPORTED, "grid too large");
    kern<<<(unsigned)grid, kThreads + 32, L::BYTES, stream>>>(tp, *map);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ACCSPMM_ERR_CUDA, std::string("tcgen05 spmm launch: ") + cudaGetErrorString(e));
    return ACCSPMM_OK;
}

}  // namespace

#ifdef ACCSPMM_VARIANTS
void debug_tc05_trace(unsigned long long *out)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_tc05_trace, sizeof(g_tc05_trace));
}
#endif

accspmm_status launch_spmm_tc05(const DevicePlan &d, const void *B, int64_t N, float *C, float *ws, uint32_t *counters,
                                void *stream, bool round_b)
{
    if (d.rows == 0 || d.n_units == 0) return ACCSPMM_OK;
    if (N % kFW != 0) return fail(ACCSPMM_ERR_INTERNAL, "tcgen05 kernel needs N % 128 == 0");
    TcParams tp;
    tp.rwo = d.rwo;
    tp.tco = d.tco;
    tp.a2b = d.a2b;
    tp.bits = d.bits;
    tp.vals = reinterpret_cast<const float *>(d.vals);
    tp.units = reinterpret_cast<const uint4 *>(d.units);
    tp.row_map = d.row_map;
    tp.C = C;
    tp.ws = ws;
    tp.counters = counters;
    tp.N = N;
    tp.rows = d.rows;
    tp.n_units = d.n_units;
    tp.nslices = (int32_t)(N / kFW);
    tp.wh = d.wh;
    tp.nw = d.wh / kWindow;
    tp.slice_major = tp.nslices > 1 ? 1 : 0;
    static const CUtensorMap no_map = {};
    const CUtensorMap *map = &no_map;  // no TC blocks (K = 0): no TMA is ever issued
    if (d.NB > 0) {
        accspmm_status st = tensor_map_tc05(d, B, N, &map);
        if (st != ACCSPMM_OK) return st;
    }
    cudaStream_t s = (cudaStream_t)stream;
#ifdef ACCSPMM_VARIANTS
    // measurement variants of the tcgen05 kernel (ACCSPMM_KCFG): wait flavour
    // (60: test_wait spin, 61: try_wait without a suspend hint) and deeper TMEM rings (62/63: SA 8)
    switch (knobs().kcfg) {
    case 60:
        if (d.wh <= 16) return round_b ? launch_tc<16, 6, 4, 2, true, 1>(tp, map, s) : launch_tc<16, 6, 4, 2, false, 1>(tp, map, s);
        return round_b ? launch_tc<32, 6, 4, 1, true, 1>(tp, map, s) : launch_tc<32, 6, 4, 1, false, 1>(tp, map, s);
    case 61:
        if (d.wh <= 16) return round_b ? launch_tc<16, 6, 4, 2, true, 2>(tp, map, s) : launch_tc<16, 6, 4, 2, false, 2>(tp, map, s);
        return round_b ? launch_tc<32, 6, 4, 1, true, 2>(tp, map, s) : launch_tc<32, 6, 4, 1, false, 2>(tp, map, s);
    case 62:
        if (d.wh <= 16) return round_b ? launch_tc<16, 8, 8, 2, true, 1>(tp, map, s) : launch_tc<16, 8, 8, 2, false, 1>(tp, map, s);
        return round_b ? launch_tc<32, 8, 8, 1, true, 1>(tp, map, s) : launch_tc<32, 8, 8, 1, false, 1>(tp, map, s);
    case 63:
        if (d.wh <= 16) return round_b ? launch_tc<16, 8, 8, 2, true, 0>(tp, map, s) : launch_tc<16, 8, 8, 2, false, 0>(tp, map, s);
        return round_b ? launch_tc<32, 8, 8, 1, true, 0>(tp, map, s) : launch_tc<32, 8, 8, 1, false, 0>(tp, map, s);
    case 64:  // one commit per 2 MMAs
        if (d.wh <= 16) return round_b ? launch_tc<16, 6, 4, 2, true, 0, 2>(tp, map, s) : launch_tc<16, 6, 4, 2, false, 0, 2>(tp, map, s);
        return round_b ? launch_tc<32, 6, 4, 1, true, 0, 2>(tp, map, s) : launch_tc<32, 6, 4, 1, false, 0, 2>(tp, map, s);
    case 65:  // one commit per 4 MMAs, 8 stages
        if (d.wh <= 16) return round_b ? launch_tc<16, 8, 8, 2, true, 0, 4>(tp, map, s) : launch_tc<16, 8, 8, 2, false, 0, 4>(tp, map, s);
        return round_b ? launch_tc<32, 8, 8, 1, true, 0, 4>(tp, map, s) : launch_tc<32, 8, 8, 1, false, 0, 4>(tp, map, s);
    case 68: {  // phase trace (g_tc05_trace; read with accspmm_debug_tc05_trace)
        void *sym = nullptr;
        cudaGetSymbolAddress(&sym, g_tc05_trace);
        cudaMemsetAsync(sym, 0, sizeof(g_tc05_trace), s);
        if (d.wh <= 16) return launch_tc<16, 6, 4, 2, false, 0, 1, 1, true>(tp, map, s);
        return launch_tc<32, 6, 4, 1, false, 0, 1, 1, true>(tp, map, s);
    }
    case 66:  // timing probe: every MMA issued twice (wrong results)
        if (d.wh <= 16) return launch_tc<16, 6, 4, 2, false, 0, 1, 2>(tp, map, s);
        return launch_tc<32, 6, 4, 1, false, 0, 1, 2>(tp, map, s);
    case 67:  // timing probe: every MMA issued four times (wrong results)
        if (d.wh <= 16) return launch_tc<16, 6, 4, 2, false, 0, 1, 4>(tp, map, s);
        return launch_tc<32, 6, 4, 1, false, 0, 1, 4>(tp, map, s);
    default: break;
    }
#endif
    // ring depths: ST gather stages (L2 latency), SA TMEM/B-tile stages (MMA latency), ND
    // accumulators (epilogue overlap for short windows); TMEM 64 columns -> 8 CTAs per SM
    if (d.wh <= 16) return round_b ? launch_tc<16, 6, 4, 2, true>(tp, map, s) : launch_tc<16, 6, 4, 2, false>(tp, map, s);
    return round_b ? launch_tc<32, 6, 4, 1, true>(tp, map, s) : launch_tc<32, 6, 4, 1, false>(tp, map, s);
}

}  // namespace accspmm
