// gather_bench2.cu — properly pipelined staging micro-benchmark (sm_100a): producer warps
// run ahead over an S-stage ring of 16 KB blocks (128 rows x 128 B, 128B-swizzled), one
// consumer warp waits/releases.  Compares TMA tile, TMA gather4 and row-coalesced cp.async
// for scattered 128 B rows, L2-resident or DRAM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2506_03275_b200/csrc scripts/gather_bench2.cu -o scripts/gather_bench2 -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace csd::tc;

constexpr int kStages = 6;
constexpr int kBlk = 128 * 128;

// row index of row `r` in block `it` (computed, not loaded: isolates the copy path)
__device__ __forceinline__ int hrow(int it, int r, int nrows) {
    uint32_t x = (uint32_t)(it * 1315423911u) ^ (uint32_t)(r * 2654435761u) ^ (blockIdx.x * 97531u);
    x ^= x >> 15;
    x *= 0x2c1b3c6du;
    x ^= x >> 12;
    return (int)(x % (uint32_t)nrows);
}

// mode 0: TMA tile (1 thread); 1: gather4 spread over producer warps; 2: cp.async coalesced
__global__ void __launch_bounds__(544, 1)
k_bench(const __grid_constant__ CUtensorMap tile_map, const __grid_constant__ CUtensorMap g4_map,
        const __nv_bfloat16* base, int ld, const int* rows, int nrows, int iters, int mode,
        int nprod, unsigned long long* sink) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kBlk);
    uint64_t* empty = full + kStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pw = nprod / 32;  // producer warps; consumer = warp pw
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + s, mode == 2 ? nprod : mode == 3 ? nprod - 31 : 1);
            mbar_init(empty + s, 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    unsigned long long acc = 0;
    if (warp < pw) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % kStages;
            const int rbase = ((blockIdx.x * 7919 + it * 131) % (nrows / 128)) * 128;
            if (it >= kStages) mbar_wait(empty + s, ((it / kStages) - 1) & 1);
            uint8_t* dst = smem + s * kBlk;
            if (mode == 0) {
                if (threadIdx.x == 0) {
                    mbar_arrive_expect_tx(full + s, kBlk);
                    tma_load_2d(&tile_map, full + s, dst, 0, rbase);
                }
            } else if (mode == 1) {
                if (threadIdx.x == 0) mbar_arrive_expect_tx(full + s, kBlk);
                for (int g = threadIdx.x; g < 32; g += nprod) {  // 32 gather4 per block
                    int r[4];
                    for (int i = 0; i < 4; ++i) r[i] = hrow(it, g * 4 + i, nrows);
                    tma_gather4(&g4_map, full + s, dst + g * 512, 0, r[0], r[1], r[2], r[3]);
                }
            } else if (mode == 3) {
                // hybrid: rows [0, 128 * frac) by gather4 from warp 0, the rest by cp.async
                // from warps 1.. (row-coalesced); full barrier: 1 (expect_tx) + cp.async threads
                const int g4rows = (int)(128 * 0.3f) & ~3;
                if (warp == 0) {
                    if (lane == 0) mbar_arrive_expect_tx(full + s, g4rows * 128);
                    for (int g = lane; g < g4rows / 4; g += 32) {
                        int r[4];
                        for (int i = 0; i < 4; ++i) r[i] = hrow(it, g * 4 + i, nrows);
                        tma_gather4(&g4_map, full + s, dst + g * 512, 0, r[0], r[1], r[2], r[3]);
                    }
                } else {
                    for (int idx = g4rows * 8 + threadIdx.x - 32; idx < 128 * 8; idx += nprod - 32) {
                        const int row = idx >> 3, c = idx & 7;
                        const uint8_t* src =
                            reinterpret_cast<const uint8_t*>(base + (size_t)hrow(it, row, nrows) * ld) + c * 16;
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst) + sw128_offset(row, c)),
                                     "l"(src));
                    }
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + s)));
                }
            } else {
                for (int idx = threadIdx.x; idx < 128 * 8; idx += nprod) {
                    const int row = idx >> 3, c = idx & 7;
                    const uint8_t* src =
                        reinterpret_cast<const uint8_t*>(base + (size_t)hrow(it, row, nrows) * ld) + c * 16;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst) + sw128_offset(row, c)),
                                 "l"(src));
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + s)));
            }
        }
    } else if (warp == pw) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % kStages;
            mbar_wait(full + s, (it / kStages) & 1);
            acc += reinterpret_cast<const uint32_t*>(smem + s * kBlk)[lane * 97];
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

int main() {
    const int rows_total = 1 << 17, ld = 3072;
    const size_t elems = (size_t)rows_total * ld;
    __nv_bfloat16* d;
    cudaMalloc(&d, elems * 2);
    cudaMemset(d, 1, elems * 2);
    std::vector<int> h(rows_total), hl(rows_total), hs(rows_total);
    srand(1);
    for (int i = 0; i < rows_total; ++i) {
        h[i] = rand() % rows_total;
        hl[i] = rand() % 16384;  // 2 MB touched: L2-resident
        hs[i] = i;
    }
    int *rows, *rows_l2;
    cudaMalloc(&rows, rows_total * 4);
    cudaMalloc(&rows_l2, rows_total * 4);
    cudaMemcpy(rows, h.data(), rows_total * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(rows_l2, hl.data(), rows_total * 4, cudaMemcpyHostToDevice);
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    CUtensorMap tm, tg;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows_total};
    cuuint64_t str[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box_t[2] = {64, 128}, box_g[2] = {64, 1}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box_t, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box_g, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int smem = kStages * kBlk + 1024 + 256;
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 3000;
    struct Case { const char* name; int mode; const int* r; int nprod; int nrows; };
    Case cases[] = {
        {"tma tile", 0, nullptr, 32, 16384},
        {"gather4 1 warp (L2)", 1, nullptr, 32, 16384},
        {"gather4 4 warps (L2)", 1, nullptr, 128, 16384},
        {"gather4 4 warps (DRAM)", 1, nullptr, 128, 1 << 17},
        {"cp.async coalesced 1 warp (L2)", 2, nullptr, 32, 16384},
        {"cp.async coalesced 2 warps (L2)", 2, nullptr, 64, 16384},
        {"cp.async coalesced 4 warps (L2)", 2, nullptr, 128, 16384},
        {"cp.async coalesced 8 warps (L2)", 2, nullptr, 256, 16384},
        {"cp.async coalesced 4 warps (DRAM)", 2, nullptr, 128, 1 << 17},
        {"hybrid 30% g4 (1 warp) + cp.async 2 warps", 3, nullptr, 96, 16384},
        {"hybrid 30% g4 (1 warp) + cp.async 3 warps", 3, nullptr, 128, 16384},
        {"cp.async coalesced 8 warps (DRAM)", 2, nullptr, 256, 1 << 17},
    };
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (const Case& cs : cases) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_bench<<<148, cs.nprod + 32, smem>>>(tm, tg, d, ld, cs.r, cs.nrows, iters, cs.mode,
                                                  cs.nprod, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep)
                printf("%-42s %8.1f GB/s  (%.1f B/ns per SM)\n", cs.name,
                       148.0 * iters * kBlk / (ms * 1e-3) / 1e9, (double)iters * kBlk / (ms * 1e6));
        }
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
