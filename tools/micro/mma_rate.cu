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

// completed-phase probe without the try_wait suspend path
__device__ __forceinline__ void mbar_wait_probe(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "PROBE_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra PROBE_%=;\n}" ::"r"(addr),
        "r"(parity)
        : "memory");
}

// sequence ids
//  0: SS M128 N32  K128          1: SS M128 N64  K128     2: SS M128 N128 K128   3: SS M128 N256 K128
//  4: TS M128 N32  K128          5: TS M128 N64  K128     6: TS M128 N128 K128
//  7: current dK/dV iteration (64 queries): S^T, dP^T SS N64 K128 ; dV, dK TS N128 K64
//  8: proposed dK/dV iteration (2 x 32 queries): S^T, dP^T TS N32 K128 ; dV, dK TS N128 K32
//  9: proposed with 64-query tiles: S^T, dP^T TS N64 K128 ; dV, dK TS N128 K64
__global__ void __launch_bounds__(128, 1) mma_rate(int seq, int iters, long long* cycles, const uint8_t* gsrc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t slot;
    __shared__ uint64_t bar, bar2, bar3;
    __shared__ volatile int flag;
    // seq 13, 14: random bf16 operands (N(0, 1)-like), else zeros
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (seq >= 13) {
            uint32_t h = (i * 2654435761u) ^ (blockIdx.x * 40503u);
            uint32_t w[4];
            for (int j = 0; j < 4; ++j) {
                h ^= h << 13; h ^= h >> 17; h ^= h << 5;
                const float a = (static_cast<float>(h & 0xffff) / 32768.f - 1.f) * 2.f;
                const float b = (static_cast<float>(h >> 16) / 32768.f - 1.f) * 2.f;
                w[j] = pack2(a, b);
            }
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        reinterpret_cast<uint4*>(sm)[i] = v;
    }
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1 << 20);  // commits arrive here and never complete a phase
        mbar_init(&bar3, 1);
        mbar_arrive(&bar3);          // phase 0 complete: waits on it return at once
        flag = 1;
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
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    const int mseq = seq == 13 ? 2 : seq >= 11 && seq <= 14 ? 10 : seq;
    __shared__ uint64_t tbar;
    if (seq == 12 && warp == 1) {
        // TMA-like bulk copies (global -> shared, 2 x 32 KB in flight) into a
        // separate region while the MMAs run: the dK/dV item's Q / dO refills
        if ((threadIdx.x & 31) == 0) {
            mbar_init(&tbar, 1);
            fence_barrier_init();
            uint32_t ph = 0;
            long long n = 0;
            while (!done) {
                mbar_expect_tx(&tbar, 65536);
                bulk_load_1d(sm + 98304, gsrc + (n & 63) * 65536, 32768, &tbar);
                bulk_load_1d(sm + 98304 + 32768, gsrc + (n & 63) * 65536 + 32768, 32768, &tbar);
                mbar_wait(&tbar, ph);
                ph ^= 1;
                ++n;
            }
            cycles[blockIdx.x + 148] = n;
        }
    }
    if (seq == 11 && warp >= 1) {
        // elementwise-like TMEM traffic on the S / dP columns while the MMAs run
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        unsigned acc = 0;
        while (!done) {
            uint32_t a[32], b[32];
            tmem_ld32(tmem + lane_off + 0, a);
            tmem_ld32(tmem + lane_off + 128, b);
            tmem_ld_wait();
            uint32_t c[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) c[j] = a[j] ^ b[j + 16];
            tmem_st16(tmem + lane_off + 64, c);
            tmem_st_wait();
            acc += c[3];
        }
        if (acc == 12345) cycles[blockIdx.x + 148] = acc;
    }
    if (threadIdx.x == 0) {
        auto kmaj = [](uint32_t base, int kk) { return umma_desc_sw128(base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024); };
        auto mn = [](uint32_t base, int kk) { return umma_desc_sw128(base + kk * 2048, 8192, 1024); };
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            switch (mseq) {
                case 0: case 1: case 2: case 3: {
                    const int n = 32 << mseq;
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
                case 10:    // round-2 dK/dV iteration (128 queries): S^T, dP^T SS N128 K128; dV, dK TS N128 K128
                case 15:    // + tcgen05.fence::after_thread_sync before each group (the kernel's pattern)
                case 16:    // + a commit to an mbarrier after each group
                case 17:    // + an mbarrier wait (already-completed phase) before each group
                case 19:    // + mbarrier.test_wait probe instead
                case 20:    // + a volatile shared-memory flag read instead
                case 18: {  // + two waits before each group
                    const uint32_t ids = umma_idesc_bf16(128, 128, false, false), idg = umma_idesc_bf16(128, 128, false, true);
                    auto sep = [&]() {
                        if (mseq == 15 || mseq == 16) tc_fence_after();
                        if (mseq == 16) tc_commit(&bar2);
                        if (mseq == 17 || mseq == 18) mbar_wait(&bar3, 0);
                        if (mseq == 18) mbar_wait(&bar3, 0);
                        if (mseq == 19) mbar_wait_probe(&bar3, 0);
                        if (mseq == 20) {
                            while (flag == 0) {
                            }
                        }
                    };
                    sep();
                    for (int kk = 0; kk < 8; ++kk) tc_mma_bf16(tmem, kmaj(a_s, kk), kmaj(b_s, kk), ids, 1);
                    sep();
                    for (int kk = 0; kk < 8; ++kk) tc_mma_bf16(tmem + 128, kmaj(a_s, kk), kmaj(c_s, kk), ids, 1);
                    sep();
                    for (int kk = 0; kk < 8; ++kk)
                        tc_mma_bf16_ts(tmem + 256, tmem + (kk >> 2) * 64 + (kk & 3) * 8, mn(b_s, kk), idg, 1);
                    sep();
                    for (int kk = 0; kk < 8; ++kk)
                        tc_mma_bf16_ts(tmem + 384, tmem + 128 + (kk >> 2) * 64 + (kk & 3) * 8, mn(c_s, kk), idg, 1);
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
        done = 1;
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
    cudaMalloc(&cyc, 2 * 148 * sizeof(long long));
    const int smem = 97 * 1024 + 1024 + 64 * 1024;
    uint8_t* gsrc;
    cudaMalloc(&gsrc, 64 << 16);
    cudaMemset(gsrc, 0, 64 << 16);
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // FLOP per round of each sequence
    const double fl[21] = {2.0 * 128 * 32 * 128,  2.0 * 128 * 64 * 128,  2.0 * 128 * 128 * 128, 2.0 * 128 * 256 * 128,
                           2.0 * 128 * 32 * 128,  2.0 * 128 * 64 * 128,  2.0 * 128 * 128 * 128,
                           4 * 2.0 * 128 * 64 * 128, 8 * 2.0 * 128 * 32 * 128, 4 * 2.0 * 128 * 64 * 128,
                           4 * 2.0 * 128 * 128 * 128, 4 * 2.0 * 128 * 128 * 128, 4 * 2.0 * 128 * 128 * 128,
                           2.0 * 128 * 128 * 128, 4 * 2.0 * 128 * 128 * 128, 4 * 2.0 * 128 * 128 * 128,
                           4 * 2.0 * 128 * 128 * 128, 4 * 2.0 * 128 * 128 * 128, 4 * 2.0 * 128 * 128 * 128,
                           4 * 2.0 * 128 * 128 * 128, 4 * 2.0 * 128 * 128 * 128};
    const char* name[21] = {"SS N32", "SS N64", "SS N128", "SS N256", "TS N32", "TS N64", "TS N128",
                            "dkdv current (SS N64 + TS N128 K64)", "dkdv proposed (TS N32 + TS N128 K32) x2",
                            "dkdv TS N64 + TS N128 K64", "dkdv r2 (SS N128 x2 + TS N128 K128 x2)",
                            "dkdv r2 + concurrent tcgen05.ld/st traffic", "dkdv r2 + concurrent bulk copies to smem",
                            "SS N128, random operands", "dkdv r2, random operands",
                            "dkdv r2 + fence::after_thread_sync per group", "dkdv r2 + fence + commit per group",
                            "dkdv r2 + completed mbarrier wait per group", "dkdv r2 + 2 completed waits per group",
                            "dkdv r2 + test_wait probe per group", "dkdv r2 + volatile smem flag read per group"};
    for (int seq = 0; seq < 21; ++seq) {
        const int iters = 2000;
        mma_rate<<<148, 128, smem>>>(seq, 20, cyc, gsrc);
        mma_rate<<<148, 128, smem>>>(seq, iters, cyc, gsrc);
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
        if (seq == 12) {
            long long hb[148];
            cudaMemcpy(hb, cyc + 148, sizeof(hb), cudaMemcpyDeviceToHost);
            double nb = 0;
            for (int i = 0; i < 148; ++i) nb += hb[i];
            printf("    bulk copies: %.1f KB per MMA round per SM\n", nb / 148 * 64.0 / iters);
        }
    }
    return 0;
}
