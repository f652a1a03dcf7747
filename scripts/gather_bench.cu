// gather_bench.cu — micro-benchmark of the three ways to stage 128 scattered 128-byte rows
// (one K/V or weight-row block) into 128B-swizzled shared memory on sm_100a:
//   mode 0: TMA 2D tile (contiguous rows; reference point)
//   mode 1: TMA tile::gather4, 32 instructions per block (one per lane)
//   mode 2: cp.async 16 B by 128 threads (8 per thread), mbarrier-tracked
// Each CTA (one per SM) streams `iters` blocks through a 4-stage ring; prints GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2506_03275_b200/csrc scripts/gather_bench.cu -o scripts/gather_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace csd::tc;

#ifndef STAGES
#define STAGES 4
#endif
constexpr int kStages = STAGES;
constexpr int kBlk = 128 * 128;

__global__ void __launch_bounds__(512, 1)
k_bench(const __grid_constant__ CUtensorMap tile_map, const __grid_constant__ CUtensorMap g4_map,
        const __nv_bfloat16* base, int ld, const int* rows, int nrows, int iters, int mode,
        unsigned long long* sink) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kBlk);
    uint64_t* empty = full + kStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + s, mode == 5 ? 128 : mode == 6 ? 65 : mode == 7 ? blockDim.x : 1);
            mbar_init(empty + s, blockDim.x / 32);
        }
        fence_barrier_init();
    }
    __syncthreads();
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int s = it % kStages;
        const int rbase = ((blockIdx.x * 7919 + it * 131) % (nrows / 128)) * 128;
        if (it >= kStages) mbar_wait(empty + s, ((it / kStages) - 1) & 1);
        uint8_t* dst = smem + s * kBlk;
        if (mode == 0) {
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(full + s, kBlk);
                tma_load_2d(&tile_map, full + s, dst, 0, rows[rbase]);
            }
        } else if (mode == 1) {
            if (warp == 0) {
                if (lane == 0) mbar_arrive_expect_tx(full + s, kBlk);
                __syncwarp();
                const int* r = rows + rbase + lane * 4;
                tma_gather4(&g4_map, full + s, dst + lane * 512, 0, r[0], r[1], r[2], r[3]);
            }
        } else if (mode == 3) {
            if (threadIdx.x == 0) mbar_arrive_expect_tx(full + s, kBlk);
            __syncthreads();
            const int nw = blockDim.x / 32, per = 32 / nw;
            if (lane < per) {  // nw warps x (32/nw) lanes x gather4
                const int g = warp * per + lane;
                const int* r = rows + rbase + g * 4;
                tma_gather4(&g4_map, full + s, dst + g * 512, 0, r[0], r[1], r[2], r[3]);
            }
        } else if (mode == 4) {
            // unswizzled staging: one 128 B bulk copy per row (layout not MMA-ready; cost probe)
            if (threadIdx.x == 0) mbar_arrive_expect_tx(full + s, kBlk);
            __syncthreads();
            const int row = threadIdx.x;
            if (row >= 128) goto consume;
            {
            const __nv_bfloat16* src = base + (size_t)rows[rbase + row] * ld;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                ::"r"(smem_u32(dst + row * 128)), "l"(src), "r"(smem_u32(full + s)) : "memory");
            }
        } else if (mode == 6) {
            // mixed: rows [0,64) by TMA gather4 (warps 0-3, 4 instructions each), rows
            // [64,128) by cp.async 16 B (threads 128..191, one row x 8 chunks each)
            if (threadIdx.x == 0) mbar_arrive_expect_tx(full + s, kBlk / 2);
            __syncthreads();
            if (warp < 4 && lane < 4) {
                const int g = warp * 4 + lane;
                const int* r = rows + rbase + g * 4;
                tma_gather4(&g4_map, full + s, dst + g * 512, 0, r[0], r[1], r[2], r[3]);
            } else if (threadIdx.x >= 128 && threadIdx.x < 192) {
                const int row = 64 + threadIdx.x - 128;
                const uint8_t* src = reinterpret_cast<const uint8_t*>(base + (size_t)rows[rbase + row] * ld);
                for (int c = 0; c < 8; ++c) {
                    const uint32_t d = smem_u32(dst) + sw128_offset(row, c);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + c * 16));
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + s)));
            }
        } else if (mode >= 8 && mode <= 10) {
            // raw 1D bulk copies of contiguous row segments (no swizzle): mode 8 = 128 B x 128
            // rows, 9 = 256 B x 64 rows, 10 = 1 KB x 16 rows (16 KB per stage in all cases)
            const int seg = mode == 8 ? 128 : mode == 9 ? 256 : 1024;
            const int nseg = kBlk / seg;
            if (threadIdx.x == 0) mbar_arrive_expect_tx(full + s, kBlk);
            __syncthreads();
            for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
                const __nv_bfloat16* src = base + (size_t)rows[rbase + i] * ld;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %3, [%2];"
                    ::"r"(smem_u32(dst + i * seg)), "l"(src), "r"(smem_u32(full + s)), "r"(seg) : "memory");
            }
        } else if (mode == 7) {
            // row-coalesced cp.async: 8 consecutive lanes fetch one row's 128 B (8 x 16 B,
            // swizzled destinations); each warp instruction covers 4 rows
            const int nthr = blockDim.x;
            for (int idx = threadIdx.x; idx < 128 * 8; idx += nthr) {
                const int row = idx >> 3, c = idx & 7;
                const uint8_t* src = reinterpret_cast<const uint8_t*>(base + (size_t)rows[rbase + row] * ld) + c * 16;
                const uint32_t d = smem_u32(dst) + sw128_offset(row, c);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + s)));
        } else {  // mode 5
            // 128 threads x 8 x 16 B; row = tid, chunks 0..7 swizzled
            const int row = threadIdx.x;
            const uint8_t* src = reinterpret_cast<const uint8_t*>(base + (size_t)rows[rbase + row] * ld);
            for (int c = 0; c < 8; ++c) {
                const uint32_t d = smem_u32(dst) + sw128_offset(row, c);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + c * 16));
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + s)));
        }
    consume:
        // consumer: every warp waits, touches one word, releases
        mbar_wait(full + s, (it / kStages) & 1);
        acc += reinterpret_cast<const uint32_t*>(dst)[threadIdx.x];
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

int main(int argc, char** argv) {
    const int g_ctas = getenv("CTAS") ? atoi(getenv("CTAS")) : 148;
    const int rows_total = 1 << 17, cols = 64;  // 128 B rows (one 64-column strip)
    const int ld = 3072;                         // real pitch: rows of a [F, 3072] weight
    const size_t elems = (size_t)rows_total * ld;
    __nv_bfloat16* d;
    cudaMalloc(&d, elems * 2);
    cudaMemset(d, 1, elems * 2);
    std::vector<int> h(rows_total);
    srand(1);
    for (int i = 0; i < rows_total; ++i) h[i] = rand() % rows_total;
    int* rows;
    cudaMalloc(&rows, rows_total * 4);
    cudaMemcpy(rows, h.data(), rows_total * 4, cudaMemcpyHostToDevice);
    std::vector<int> seq(rows_total);
    for (int i = 0; i < rows_total; ++i) seq[i] = i;
    int* rows_seq;
    cudaMalloc(&rows_seq, rows_total * 4);
    cudaMemcpy(rows_seq, seq.data(), rows_total * 4, cudaMemcpyHostToDevice);
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    CUtensorMap tm, tg;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows_total};
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
    const int iters = 2000;
    // rows restricted to the first `l2rows` rows for the L2-resident variants
    const int l2rows = 16384;  // 16384 x 6 KB pitch: 100 MB span, but only 2 MB touched
    std::vector<int> hl(rows_total);
    for (int i = 0; i < rows_total; ++i) hl[i] = rand() % l2rows;
    int* rows_l2;
    cudaMalloc(&rows_l2, rows_total * 4);
    cudaMemcpy(rows_l2, hl.data(), rows_total * 4, cudaMemcpyHostToDevice);
    struct Case { const char* name; int mode; const int* r; int threads; };
    Case cases[] = {
        {"tma tile (contiguous rows)", 0, rows_seq, 128},
        {"tma gather4 1 warp (random, L2)", 1, rows_l2, 128},
        {"tma gather4 4 warps x8 (random, L2)", 3, rows_l2, 128},
        {"tma gather4 8 warps x4 (random, L2)", 3, rows_l2, 256},
        {"tma gather4 16 warps x2 (random, L2)", 3, rows_l2, 512},
        {"tma gather4 8 warps x4 (random, DRAM)", 3, rows, 256},
        {"tma gather4 16 warps x2 (random, DRAM)", 3, rows, 512},
        {"bulk 1D 128 B segments (L2)", 8, rows_l2, 128},
        {"bulk 1D 256 B segments (L2)", 9, rows_l2, 128},
        {"bulk 1D 1 KB segments (L2)", 10, rows_l2, 128},
        {"bulk 1D 256 B segments (DRAM)", 9, rows, 128},
        {"bulk 1D 1 KB segments (DRAM)", 10, rows, 128},
        {"cp.async row-coalesced 128 thr (L2)", 7, rows_l2, 128},
        {"cp.async row-coalesced 256 thr (L2)", 7, rows_l2, 256},
        {"cp.async row-coalesced 512 thr (L2)", 7, rows_l2, 512},
        {"cp.async row-coalesced 256 thr (DRAM)", 7, rows, 256},
        {"cp.async 128 thr (random, L2)", 5, rows_l2, 128},
        {"cp.async 128 thr (random, DRAM)", 5, rows, 128},
        {"mixed g4 4 warps + cp.async 64 thr (L2)", 6, rows_l2, 256},
        {"mixed g4 4 warps + cp.async 64 thr (DRAM)", 6, rows, 256},
    };
    for (const Case& cs : cases) {
        const int mode = cs.mode;
        const int* r = cs.r;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            k_bench<<<g_ctas, cs.threads, smem>>>(tm, tg, d, ld, r, rows_total, iters, mode, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double bytes = (double)g_ctas * iters * kBlk;
            if (rep) printf("%-38s %8.3f ms  %8.1f GB/s  (%.0f ns per 16 KB block per SM)\n", cs.name, ms,
                            bytes / (ms * 1e-3) / 1e9, ms * 1e6 / iters);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
