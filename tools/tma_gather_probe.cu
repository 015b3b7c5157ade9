// TMA tile::gather4 throughput probe (measurement tool, not product code).
//
// Question it answers (DESIGN.md §6/§10): how many bytes per SM cycle can cp.async.bulk.tensor
// .2d.tile::gather4 deliver from an L2-resident B as a function of the box width (bytes per
// gathered row), the swizzle mode and the number of requests in flight per SM?  A tcgen05 SS
// design needs the gathered rows in the MN-major SW128 layout: 32 TF32 features (128 B) per
// request row, i.e. 8 gather4 per 8x8 block at 128 features instead of 2 of 544 B today.
//
// Each CTA = 1 warp; lane 0 keeps `stages` stages in flight, each stage = `reqs` gather4 of
// random rows (precomputed row ids), and waits on the oldest stage's mbarrier before
// re-issuing it.  No consumer work: this is the producer-side ceiling.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_gather_probe tools/tma_gather_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));         \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32) probe_kernel(const __grid_constant__ CUtensorMap map, const int32_t *__restrict__ rows,
                                                   int64_t nrows_idx, int iters, int stages, int reqs, int box_bytes,
                                                   int col_step, int ncolgroups, unsigned long long *sink)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    uint8_t *data = smem + 1024;
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[s])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    if (lane != 0) return;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    const uint32_t stage_bytes = (uint32_t)reqs * 4u * (uint32_t)box_bytes;
    // row ids from a counter hash (no dependent index loads in the issue loop)
    // per-CTA start and odd stride (a shared stride made CTA b + 1 request CTA b's rows one step
    // later, so all SMs hit the same L2 lines at once; results before this fix understate the rate)
    auto mix = [](uint32_t h) { h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16; return h; };
    uint32_t ctr = mix(blockIdx.x * 2u + 1u);
    const uint32_t stride = mix(blockIdx.x ^ 0x5bd1e995u) | 1u;
    const uint32_t K = (uint32_t)nrows_idx;
    auto next_row = [&]() -> int32_t {
        uint32_t h = (ctr += stride);
        h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
        return (int32_t)__umulhi(h, K);
    };
    int32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
    auto issue = [&](int s) {
        const uint32_t b = smem_u32(&bar[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(stage_bytes) : "memory");
        const uint32_t dst0 = smem_u32(data + (size_t)s * stage_bytes);
        for (int q = 0; q < reqs; ++q) {
            // ncolgroups > 1: the requests of one group of rows walk the column groups (the
            // SW128 pattern: the same 4 rows, 32 features each, 4 times)
            const int cg = q % ncolgroups;
            if (cg == 0) { r0 = next_row(); r1 = next_row(); r2 = next_row(); r3 = next_row(); }
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n" ::"r"(dst0 + (uint32_t)q * 4u * (uint32_t)box_bytes),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(cg * col_step), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b),
                "l"(pol)
                : "memory");
        }
    };
    for (int s = 0; s < stages; ++s) issue(s);
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int s = it % stages;
        const uint32_t ph = (uint32_t)(it / stages) & 1u;
        asm volatile(
            "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@P1 bra D_%=;\n\tbra W_%=;\n\tD_%=:\n\t}\n" ::"r"(smem_u32(&bar[s])),
            "r"(ph)
            : "memory");
        acc += data[(size_t)s * stage_bytes + (it & 63)];
        if (it + stages < iters) issue(s);
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

int main(int argc, char **argv)
{
    const int64_t K = 232965;  // Reddit-shaped rows
    const int64_t N = 128;     // TF32 features per row
    float *B;
    CK(cudaMalloc(&B, K * N * 4));
    CK(cudaMemset(B, 0, K * N * 4));
    const int64_t nidx = 1 << 22;
    std::vector<int32_t> h(nidx);
    uint64_t x = 88172645463325252ull;
    for (int64_t i = 0; i < nidx; ++i) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        h[i] = (int32_t)(x % (uint64_t)K);
    }
    int32_t *rows;
    CK(cudaMalloc(&rows, nidx * 4));
    CK(cudaMemcpy(rows, h.data(), nidx * 4, cudaMemcpyHostToDevice));
    unsigned long long *sink;
    CK(cudaMalloc(&sink, 8));

    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q));
    int dev = 0, sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));

    struct Case {
        const char *name;
        int box;       // elements per gathered row
        int swz;       // 0 none, 3 = 128B
        int reqs;      // gather4 per stage
        int ncg;       // column groups walked by the requests of a stage
    };
    const Case cases[] = {
        {"box136_none_2req(today TF32 N=128)", 136, 0, 2, 1},
        {"box128_none_2req", 128, 0, 2, 1},
        {"box32_none_8req", 32, 0, 8, 4},
        {"box32_sw128_8req(UMMA MN-major SW128)", 32, 3, 8, 4},
        {"box64_none_4req", 64, 0, 4, 2},
        {"box24_none_2req(today TF32 N=16)", 24, 0, 2, 1},
        {"box72_none_2req(FP16-like bytes 288)", 72, 0, 2, 1},
    };
    const int ctas_per_sm[] = {4, 8, 16, 24, 32};
    const int stage_opts[] = {2, 4};
    printf("sms %d clock_khz %d\n", sms, clk);
    for (const Case &c : cases) {
        CUtensorMap map;
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
        cuuint64_t strides[1] = {(cuuint64_t)N * 4};
        cuuint32_t box[2] = {(cuuint32_t)c.box, 1u};
        cuuint32_t estr[2] = {1u, 1u};
        CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, B, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            c.swz == 3 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("%s: encode failed %d\n", c.name, (int)r);
            continue;
        }
        const int box_bytes = c.box * 4;
        for (int st : stage_opts) {
            for (int cps : ctas_per_sm) {
                const size_t smem = 1024 + (size_t)st * c.reqs * 4 * box_bytes;
                if (smem * cps > 220 * 1024) continue;
                const int grid = sms * cps;
                const int iters = 2000;
                cudaEvent_t e0, e1;
                CK(cudaEventCreate(&e0));
                CK(cudaEventCreate(&e1));
                probe_kernel<<<grid, 32, smem>>>(map, rows, K, 50, st, c.reqs, box_bytes, 32, c.ncg, sink);
                CK(cudaGetLastError());
                CK(cudaDeviceSynchronize());
                CK(cudaEventRecord(e0));
                probe_kernel<<<grid, 32, smem>>>(map, rows, K, iters, st, c.reqs, box_bytes, 32, c.ncg, sink);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                const double req = (double)grid * iters * c.reqs;
                const double bytes = req * 4 * box_bytes;
                const double cyc = ms * 1e-3 * clk * 1e3;
                printf("%-40s stages %d ctas/SM %2d  %7.3f ms  %7.1f GB/s  %6.1f B/cyc/SM  %6.2f cyc/req/SM\n", c.name, st,
                       cps, ms, bytes / ms / 1e6, bytes / cyc / sms, cyc * sms / req);
                CK(cudaEventDestroy(e0));
                CK(cudaEventDestroy(e1));
            }
        }
    }
    return 0;
}
