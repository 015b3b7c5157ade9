// TMA gather4 ring probe (measurement tool, not product code).
//
// Question (DESIGN.md §7/§10): what puts the gather ring into the 2-4x slow mode seen with some
// layouts (stage barriers in separate 16-byte granules, 3-stage rings, one launch bound of the
// L64 layout) and once with the default kernel under ncu?  Each CTA = 1 warp running the SpMM
// kernel's ring without the math: an elected lane issues `reqs` gather4 (4 random rows of an
// L2-resident Reddit-shaped B each) per stage into a `stages`-deep ring, the warp waits on the
// oldest stage's mbarrier, optionally reads the whole stage with LDS.128 (as the MMA fragments
// do), and re-issues it.  Parameters varied one at a time: barrier placement (after the stages
// like the kernel / at the head / one 16-byte granule each), stages, CTAs per SM, the fraction of
// out-of-bounds (zero-filled padding) rows, the consumer's shared-memory reads.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_ring_probe tools/tma_ring_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));         \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Cfg {
    int stages, reqs, box_bytes, grp_bytes;  // grp = one gather4's slot (4 rows, 128-aligned)
    int bar_mode;                            // 0 after the stages (packed), 1 at the head, 2 one granule each
    int oob_per8;                            // rows out of bounds (-1) per 8 gathered rows
    int consume;                             // 0: touch one byte, 1: LDS.128 over the stage like the MMA fragments
    int iters;
    uint32_t range;                          // rows drawn from [base, base + range) (base per CTA)
    int pattern;                             // 0 random, 1 four consecutive rows per gather4, 2 stride 64 rows
};

__global__ void __launch_bounds__(32) ring_kernel(const __grid_constant__ CUtensorMap map, uint32_t K, Cfg c,
                                                  unsigned long long *sink)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    const int lane = threadIdx.x;
    const uint32_t stage_bytes = (uint32_t)c.reqs * (uint32_t)c.grp_bytes;
    const uint32_t data_bytes = stage_bytes * (uint32_t)c.stages;
    uint8_t *data = smem + (c.bar_mode == 1 ? 128 : 0);
    uint64_t *bar = reinterpret_cast<uint64_t *>(c.bar_mode == 1 ? smem : smem + ((data_bytes + 15) & ~15u));
    const int bstride = c.bar_mode == 2 ? 2 : 1;
    if (lane == 0) {
        for (int s = 0; s < c.stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[s * bstride])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    // per-CTA counter start and odd stride: CTAs draw unrelated row sequences (with a shared
    // stride, CTA b + 1 would request CTA b's rows one step later and every SM would hammer the
    // same L2 lines at once -- the flaw of the first version of this probe)
    auto mix = [](uint32_t h) { h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16; return h; };
    uint32_t ctr = mix(blockIdx.x * 2u + 1u);
    const uint32_t stride = mix(blockIdx.x ^ 0x5bd1e995u) | 1u;
    uint32_t nrow = 0;
    auto next_row = [&]() -> int32_t {
        uint32_t h = (ctr += stride);
        h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
        const bool oob = (int)(nrow++ & 7u) < c.oob_per8;
        const uint32_t base = c.range < K ? (uint32_t)(((uint64_t)blockIdx.x * 2654435761ull) % (K - c.range)) : 0u;
        return oob ? -1 : (int32_t)(base + __umulhi(h, c.range < K ? c.range : K));
    };
    auto issue = [&](int s) {
        if (lane != 0) return;
        const uint32_t b = smem_u32(&bar[s * bstride]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b),
                     "r"((uint32_t)c.reqs * 4u * (uint32_t)c.box_bytes)
                     : "memory");
        const uint32_t dst0 = smem_u32(data + (size_t)s * stage_bytes);
        for (int q = 0; q < c.reqs; ++q) {
            int32_t r0 = next_row(), r1 = next_row(), r2 = next_row(), r3 = next_row();
            if (c.pattern == 1 && r0 >= 0 && r0 + 3 < (int32_t)K) { r1 = r0 + 1; r2 = r0 + 2; r3 = r0 + 3; }
            if (c.pattern == 2 && r0 >= 0 && r0 + 192 < (int32_t)K) { r1 = r0 + 64; r2 = r0 + 128; r3 = r0 + 192; }
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n" ::"r"(dst0 + (uint32_t)q * (uint32_t)c.grp_bytes),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b), "l"(pol)
                : "memory");
        }
    };
    for (int s = 0; s < c.stages; ++s) issue(s);
    uint32_t acc = 0;
    for (int it = 0; it < c.iters; ++it) {
        const int s = it % c.stages;
        const uint32_t ph = (uint32_t)(it / c.stages) & 1u;
        asm volatile(
            "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
            "@P1 bra D_%=;\n\tbra W_%=;\n\tD_%=:\n\t}\n" ::"r"(smem_u32(&bar[s * bstride])),
            "r"(ph), "r"(0x989680)
            : "memory");
        const uint8_t *st = data + (size_t)s * stage_bytes;
        if (c.consume) {
            // the TF32 N = 128 fragment pattern: lane (g, t) reads row t of each gather, 16 B at 16 g + 128 j
            const int g = lane >> 2, t = lane & 3;
            for (int q = 0; q < c.reqs; ++q)
                for (int j = 0; j < c.box_bytes / 128; ++j) {
                    const uint4 v = *reinterpret_cast<const uint4 *>(st + q * c.grp_bytes + t * c.box_bytes + 128 * j + 16 * g);
                    acc ^= v.x ^ v.y ^ v.z ^ v.w;
                }
        } else {
            acc ^= st[(it & 63)];
        }
        __syncwarp();
        if (it + c.stages < c.iters) issue(s);
    }
    if (acc == 0x12345679u) sink[0] = acc;
}

int main()
{
    const int64_t K = 232965, N = 128;  // Reddit-shaped TF32 B (119 MB, L2-resident)
    float *B;
    CK(cudaMalloc(&B, K * N * 4));
    CK(cudaMemset(B, 0, K * N * 4));
    unsigned long long *sink;
    CK(cudaMalloc(&sink, 8));
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q));
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    printf("sms %d clock_khz %d\n", sms, clk);

    // TF32 N = 128 (box 136 = 544 B, stage 4352 B) and N = 64 (box 72 = 288 B, stage 2304 B)
    struct Case2 { const char *name; int box_el, stages, ctas, bar_mode, oob, consume; uint32_t range; int pattern; };
    const Case2 cases[] = {
        {"N128 random all K", 136, 2, 20, 0, 1, 1, 1u << 30, 0},
        {"N128 random 1/8 K", 136, 2, 20, 0, 1, 1, 29120, 0},
        {"N128 random 4096 rows", 136, 2, 20, 0, 1, 1, 4096, 0},
        {"N128 random 512 rows", 136, 2, 20, 0, 1, 1, 512, 0},
        {"N128 consecutive x4", 136, 2, 20, 0, 0, 1, 1u << 30, 1},
        {"N128 stride-64 x4", 136, 2, 20, 0, 0, 1, 1u << 30, 2},
        {"N64 random all K", 72, 2, 24, 0, 1, 1, 1u << 30, 0},
        {"N64 random 4096 rows", 72, 2, 24, 0, 1, 1, 4096, 0},
        {"N64 consecutive x4", 72, 2, 24, 0, 0, 1, 1u << 30, 1},
        {"N64 3 st 4096 rows", 72, 3, 24, 0, 1, 1, 4096, 0},
    };
    CUtensorMap maps[2];
    const int boxes[2] = {136, 72};
    for (int m = 0; m < 2; ++m) {
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
        cuuint64_t strides[1] = {(cuuint64_t)N * 4};
        cuuint32_t box[2] = {(cuuint32_t)boxes[m], 1u};
        cuuint32_t estr[2] = {1u, 1u};
        CUresult r = encode(&maps[m], CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, B, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", (int)r);
            return 1;
        }
    }
    for (int rep = 0; rep < 2; ++rep) {
        for (const Case2 &cs : cases) {
            Cfg c;
            c.stages = cs.stages;
            c.reqs = 2;
            c.box_bytes = cs.box_el * 4;
            c.grp_bytes = (4 * c.box_bytes + 127) / 128 * 128;
            c.bar_mode = cs.bar_mode;
            c.oob_per8 = cs.oob;
            c.consume = cs.consume;
            c.iters = 3000;
            c.range = cs.range;
            c.pattern = cs.pattern;
            const size_t smem = 128 + (size_t)c.stages * c.reqs * c.grp_bytes + 64;
            const CUtensorMap &map = maps[cs.box_el == 136 ? 0 : 1];
            const int grid = sms * cs.ctas;
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            Cfg w = c;  // warm-up launch
            w.iters = 100;
            ring_kernel<<<grid, 32, smem>>>(map, (uint32_t)K, w, sink);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0));
            ring_kernel<<<grid, 32, smem>>>(map, (uint32_t)K, c, sink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double req = (double)grid * c.iters * c.reqs;
            const double bytes = req * 4 * c.box_bytes;
            const double cyc = ms * 1e-3 * clk * 1e3;
            printf("rep %d %-24s st %d ctas/SM %2d bar %d oob %d lds %d  %7.3f ms %8.1f GB/s %6.2f cyc/req/SM\n", rep,
                   cs.name, cs.stages, cs.ctas, cs.bar_mode, cs.oob, cs.consume, ms, bytes / ms / 1e6, cyc * sms / req);
            CK(cudaEventDestroy(e0));
            CK(cudaEventDestroy(e1));
        }
    }
    return 0;
}
