// mma_bench.cu — tcgen05.mma issue-to-completion rate on one SM, operands resident in smem /
// TMEM (no loads, no softmax): the ceiling the attention kernel's per-block MMA chain is
// measured against.  All 148 SMs run the same loop; cycles per
// instruction and per M128·N128·K16-equivalent are printed per mode.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2506_03275_b200/csrc scripts/mma_bench.cu -o scripts/mma_bench
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace csd::tc;

// mode 0: SS M128 N128 (S = Q K^T shape, both K-major)
// mode 1: TS M128 N128 (P.V shape: A from TMEM, B MN-major in smem)
// mode 2: SS M128 N256
// mode 3: SS M128 N64
// mode 4: SS M128 N128 with B MN-major
// mode 5: mode 0 and mode 1 alternating in groups of 8 (the attention chain's mix)
// mode 6: mode 5 while 8 other warps run an ex2 / FFMA loop (softmax-like ALU load)
// mode 7: mode 5 while 8 other warps run an FFMA-only loop
// mode 8: mode 5 while 8 other warps run shuffles
// mode 9: mode 0 (SS, smem-bandwidth-bound) while 8 warps stream 16-byte smem stores
// mode 10: mode 1 (TS) while 8 warps stream 16-byte smem stores
// mode 11: mode 5 while 8 warps stream TMEM loads + stores on other columns (softmax-like)
// mode 12: mode 5 while 8 warps load / store the columns the MMAs use (as the softmax does)
// modes 13-17: SS with other M / N (the sparse MLP's tile shapes): M64 N128, M128 N144,
//              M64 N144, M128 N192, M64 N192
template <int MODE>
__global__ void __launch_bounds__(384, 1) k_mma_rate(long long* out, int groups) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
        stop = 0;
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t sA = smem_u32(smem), sB = sA + 32768;  // A: 128 x 128 bf16, B: up to 256 x 128
    constexpr uint32_t kStrip = 128 * 128;
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        const uint32_t n = MODE == 2 ? 256 : MODE == 3 ? 64 : (MODE == 14 || MODE == 15) ? 144
                         : (MODE == 16 || MODE == 17) ? 192 : 128;
        const uint32_t m = (MODE == 13 || MODE == 15 || MODE == 17) ? 64 : 128;
        const uint32_t idSS = idesc_bf16(m, n, false, false);
        const uint32_t idSSmn = idesc_bf16(128, 128, false, true);
        uint64_t da[8], db[8], dbm[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            da[kk] = desc_kmajor_sw128(sA + (kk / 4) * kStrip + (kk % 4) * 32);
            db[kk] = desc_kmajor_sw128(sB + (kk / 4) * (n * 128) + (kk % 4) * 32);
            dbm[kk] = desc_mnmajor_sw128(sB + kk * 2048, kStrip);
        }
        __syncwarp();
        t0 = clock64();
        for (int g = 0; g < groups; ++g) {
            const bool pv = MODE == 1 || MODE == 10 || ((MODE >= 5 && MODE <= 8 || MODE >= 11) && (g & 1));
            if (elect_one()) {
                if (pv) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16_ts(tmem + 256, tmem + kk * 8, dbm[kk], idSSmn, kk > 0 ? 1u : 0u);
                } else if (MODE == 4) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) mma_bf16(tmem, da[kk], dbm[kk], idSSmn, kk > 0 ? 1u : 0u);
                } else {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) mma_bf16(tmem, da[kk], db[kk], idSS, kk > 0 ? 1u : 0u);
                }
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        t1 = clock64();
        if (lane == 0) stop = 1;
    } else if (warp >= 4 && MODE >= 11) {
        const uint32_t col = MODE == 11 ? 128u + (warp >> 2) * 64u : (uint32_t)(warp >> 2) * 64u;
        const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + col;
        uint32_t acc = 0;
        while (!stop) {
            uint32_t r[32];
            tmem_ld32(ta, r);
            tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) pk[q] = r[2 * q] ^ r[2 * q + 1];
            if (MODE == 11) tmem_st16(ta + 32, pk);
            tmem_st_wait();
            acc ^= pk[3];
        }
        if (acc == 77u) out[1] = 1;
    } else if (warp >= 4 && MODE >= 9) {
        // smem write stream into the region past the operands (96 KB .. 160 KB)
        uint4* dst = reinterpret_cast<uint4*>(smem + 96 * 1024);
        const uint4 v = make_uint4(threadIdx.x, 1u, 2u, 3u);
        int i = threadIdx.x - 128;
        while (!stop) {
#pragma unroll 8
            for (int r = 0; r < 64; ++r) {
                dst[i] = v;
                i = (i + 256) & 4095;
            }
        }
    } else if (warp >= 4 && MODE >= 6) {
        float a = 0.001f * threadIdx.x, b = 1.0001f, c2 = 0.5f;
        uint32_t u = threadIdx.x;
        while (!stop) {
#pragma unroll 8
            for (int i = 0; i < 64; ++i) {
                if (MODE == 6) {
                    a = ex2_approx(fmaf(a, b, -c2));
                } else if (MODE == 7) {
                    a = fmaf(a, b, c2);
                } else {
                    u = __shfl_xor_sync(0xffffffffu, u + 1u, (i & 15) + 1);
                }
            }
        }
        if (a == 1234.5f || u == 77u) out[1] = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
        if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    }
}

template <int MODE>
static void run(const char* name, long long* d, double flop_per_instr) {
    const int groups = 2000;
    const int smem = 160 * 1024 + 1024;
    cudaFuncSetAttribute(k_mma_rate<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) k_mma_rate<MODE><<<148, 384, smem>>>(d, groups);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / (groups * 8.0);
    const double base = 128.0 * 128 * 16 * 2;
    printf("%-44s %6.1f cyc/instr  %6.1f cyc per M128N128K16-equivalent\n", name, per,
           per * base / flop_per_instr);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    const double f128 = 128.0 * 128 * 16 * 2;
    run<0>("SS M128 N128 K16 (S shape)", d, f128);
    run<1>("TS M128 N128 K16 (P.V shape, A in TMEM)", d, f128);
    run<2>("SS M128 N256 K16", d, 2 * f128);
    run<3>("SS M128 N64 K16", d, f128 / 2);
    run<4>("SS M128 N128 K16, B MN-major", d, f128);
    run<5>("S / P.V groups alternating", d, f128);
    run<6>("  ... + 8 warps ex2/FFMA loop", d, f128);
    run<7>("  ... + 8 warps FFMA loop", d, f128);
    run<8>("  ... + 8 warps shuffle loop", d, f128);
    run<9>("SS + 8 warps streaming smem stores", d, f128);
    run<10>("TS + 8 warps streaming smem stores", d, f128);
    run<11>("S/PV + 8 warps TMEM ld/st on other columns", d, f128);
    run<12>("S/PV + 8 warps TMEM loads of the MMA columns", d, f128);
    run<13>("SS M64 N128 K16", d, f128 / 2);
    run<14>("SS M128 N144 K16", d, f128 * 144 / 128);
    run<15>("SS M64 N144 K16", d, f128 * 144 / 256);
    run<16>("SS M128 N192 K16", d, f128 * 192 / 128);
    run<17>("SS M64 N192 K16", d, f128 * 192 / 256);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
