// Microbenchmark (tooling, not product): tcgen05.mma issue-limited throughput
// per SM for the shapes the attention backward uses. One CTA per SM, one
// thread issues `iters` rounds of a fixed MMA sequence into TMEM, then commits
// and waits; cycles by clock64 around the loop. Operand data is zero (rates do
// not depend on it). Prints FLOP/cycle/SM per sequence (8192 = dense peak).
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2411_15871_b200/csrc/cuda -I include tools/micro/mma_rate.cu -o /tmp/mma_rate -lcuda
#include <cstdio>

#include "common.cuh"

using namespace dh;

// sequence ids
//  0: SS M128 N32  K128          1: SS M128 N64  K128     2: SS M128 N128 K128   3: SS M128 N256 K128
//  4: TS M128 N32  K128          5: TS M128 N64  K128     6: TS M128 N128 K128
//  7: current dK/dV iteration (64 queries): S^T, dP^T SS N64 K128 ; dV, dK TS N128 K64
//  8: proposed dK/dV iteration (2 x 32 queries): S^T, dP^T TS N32 K128 ; dV, dK TS N128 K32
//  9: proposed with 64-query tiles: S^T, dP^T TS N64 K128 ; dV, dK TS N128 K64
__global__ void __launch_bounds__(128, 1) mma_rate(int seq, int iters, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t a_s = smem_u32(sm), b_s = smem_u32(sm + 32768), c_s = smem_u32(sm + 65536);
    // TMEM: D0 cols [0,128), D1 [128,256), A0 [256,320), A1 [320,384), D2 [384, 512)
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        auto kmaj = [](uint32_t base, int kk) { return umma_desc_sw128(base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024); };
        auto mn = [](uint32_t base, int kk) { return umma_desc_sw128(base + kk * 2048, 8192, 1024); };
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            switch (seq) {
                case 0: case 1: case 2: case 3: {
                    const int n = 32 << seq;
                    const uint32_t id = umma_idesc_bf16(128, n, false, false);
                    for (int kk = 0; kk < 8; ++kk) tc_mma_bf16(tmem, kmaj(a_s, kk), kmaj(b_s, kk), id, 1);
                    break;
                }
                case 4: case 5: case 6: {
                    const int n = 32 << (seq - 4);
                    const uint32_t id = umma_idesc_bf16(128, n, false, false);
                    for (int kk = 0; kk < 8; ++kk) tc_mma_bf16_ts(tmem, tmem + 256 + kk * 8, kmaj(b_s, kk), id, 1);
                    break;
                }
                case 7: {
                    const uint32_t ids = umma_idesc_bf16(128, 64, false, false), idg = umma_idesc_bf16(128, 128, false, true);
                    for (int kk = 0; kk < 8; ++kk) {
                        tc_mma_bf16(tmem, kmaj(a_s, kk), kmaj(b_s, kk), ids, 1);
                        tc_mma_bf16(tmem + 64, kmaj(a_s, kk), kmaj(c_s, kk), ids, 1);
                    }
                    for (int kk = 0; kk < 4; ++kk) {
                        tc_mma_bf16_ts(tmem + 128, tmem + kk * 8, mn(b_s, kk), idg, 1);
                        tc_mma_bf16_ts(tmem + 384, tmem + 64 + kk * 8, mn(c_s, kk), idg, 1);
                    }
                    break;
                }
                case 8: {
                    const uint32_t ids = umma_idesc_bf16(128, 32, false, false), idg = umma_idesc_bf16(128, 128, false, true);
                    for (int h = 0; h < 2; ++h) {
                        for (int kk = 0; kk < 8; ++kk) {
                            tc_mma_bf16_ts(tmem + h * 32, tmem + 256 + kk * 8, kmaj(b_s, kk), ids, 1);
                            tc_mma_bf16_ts(tmem + 64 + h * 32, tmem + 320 + kk * 8, kmaj(c_s, kk), ids, 1);
                        }
                        for (int kk = 0; kk < 2; ++kk) {
                            tc_mma_bf16_ts(tmem + 128, tmem + h * 32 + kk * 8, mn(b_s, kk), idg, 1);
                            tc_mma_bf16_ts(tmem + 384, tmem + 64 + h * 32 + kk * 8, mn(c_s, kk), idg, 1);
                        }
                    }
                    break;
                }
                case 9: {
                    const uint32_t ids = umma_idesc_bf16(128, 64, false, false), idg = umma_idesc_bf16(128, 128, false, true);
                    for (int kk = 0; kk < 8; ++kk) {
                        tc_mma_bf16_ts(tmem, tmem + 256 + kk * 8, kmaj(b_s, kk), ids, 1);
                        tc_mma_bf16_ts(tmem + 64, tmem + 320 + kk * 8, kmaj(c_s, kk), ids, 1);
                    }
                    for (int kk = 0; kk < 4; ++kk) {
                        tc_mma_bf16_ts(tmem + 128, tmem + kk * 8, mn(b_s, kk), idg, 1);
                        tc_mma_bf16_ts(tmem + 384, tmem + 64 + kk * 8, mn(c_s, kk), idg, 1);
                    }
                    break;
                }
            }
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int main() {
    long long* cyc;
    cudaMalloc(&cyc, 148 * sizeof(long long));
    const int smem = 97 * 1024 + 1024;
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // FLOP per round of each sequence
    const double fl[10] = {2.0 * 128 * 32 * 128,  2.0 * 128 * 64 * 128,  2.0 * 128 * 128 * 128, 2.0 * 128 * 256 * 128,
                           2.0 * 128 * 32 * 128,  2.0 * 128 * 64 * 128,  2.0 * 128 * 128 * 128,
                           4 * 2.0 * 128 * 64 * 128, 8 * 2.0 * 128 * 32 * 128, 4 * 2.0 * 128 * 64 * 128};
    const char* name[10] = {"SS N32", "SS N64", "SS N128", "SS N256", "TS N32", "TS N64", "TS N128",
                            "dkdv current (SS N64 + TS N128 K64)", "dkdv proposed (TS N32 + TS N128 K32) x2",
                            "dkdv TS N64 + TS N128 K64"};
    for (int seq = 0; seq < 10; ++seq) {
        const int iters = 2000;
        mma_rate<<<148, 128, smem>>>(seq, 20, cyc);
        mma_rate<<<148, 128, smem>>>(seq, iters, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
        }
        long long h[148];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        printf("%-44s %8.0f cycles/round  %7.0f FLOP/cycle/SM  (%.2f of 8192)\n", name[seq], avg / iters,
               fl[seq] * iters / avg, fl[seq] * iters / avg / 8192);
    }
    return 0;
}
