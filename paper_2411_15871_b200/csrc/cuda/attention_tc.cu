// Causal GQA flash attention on tcgen05 / TMEM / TMA (head_dim 128) — the
// attn node (forward). Replaces the mma.sync path of attention.cu for D=128.
//
// One CTA per (128-query block, q head); KV blocks of 128 keys, causal blocks
// only, heaviest query blocks first.
//   warp 0       TMA producer: Q once, K/V through a 2-stage ring
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5   softmax: thread = query row (its TMEM lane)
// TMEM (512 cols): S double buffer (2 x 128) + O accumulator (128).
//   S_j = Q K_j^T            M128 N128 K128, A=Q (K-major), B=K (K-major)
//   O  += P_j V_j            M128 N128 K128, A=P (smem, K-major), B=V (MN-major)
// The same smem tile of K/V rows serves as K-major B for QK^T and as MN-major
// B for PV (only the descriptor differs). The MMA warp issues S_{j+1} while the
// softmax warps work on S_j. Online softmax uses lazy rescaling: O (in TMEM) is
// only rescaled when a row maximum grows by more than 2^8, so the tcgen05.ld/st
// round trip is rare; P values are bounded by 2^8 in between.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "dh_capi.h"

namespace dh {
namespace {

constexpr int D = 128;
constexpr int BQ = 128;
constexpr int BKV = 128;
constexpr int kThreads = 192;
constexpr int kTile = BQ * D * 2;       // 32 KB: [2 d-halves][128 rows][128 B]
constexpr int kHalf = kTile / 2;        // 16 KB
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.f;  // log2 units

struct FwdSmem {
    // offsets from the 1024-aligned base
    static constexpr int q = 0;
    static constexpr int k = q + kTile;          // 2 stages
    static constexpr int v = k + 2 * kTile;      // 2 stages
    static constexpr int p = v + 2 * kTile;
    static constexpr int bars = p + kTile;
    static constexpr int total = bars + 256 + 1024;
};

struct FwdParams {
    float* lse;
    __nv_bfloat16* o;
    long long ldo;
    int T;
    int group;
    float scale_log2;
};

// K-major operand, 2 swizzle atoms along K (d or keys): k-step kk of 16.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int kk) {
    return umma_desc_sw128(base + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
}
// MN-major operand (V as B with N = d): k-step kk of 16 keys.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int kk) {
    return umma_desc_sw128(base + kk * 2048, kHalf, 1024);
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const FwdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + FwdSmem::bars);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;   // [2]
    uint64_t* kv_empty = bars + 3;  // [2]
    uint64_t* s_full = bars + 5;    // [2]
    uint64_t* p_full = bars + 7;
    uint64_t* pv_done = bars + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

    const int qb = gridDim.x - 1 - blockIdx.x;
    const int h = blockIdx.y;
    const int kvh = h / p.group;
    const int n_kv = qb + 1;  // causal, BQ == BKV
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&s_full[i], 1);
        }
        mbar_init(p_full, 128);
        mbar_init(pv_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t t_s0 = tmem, t_o = tmem + 256;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(q_full, kTile);
            tma_load_2d(sm + FwdSmem::q, &tm_q, q_full, h * D, qb * BQ);
            tma_load_2d(sm + FwdSmem::q + kHalf, &tm_q, q_full, h * D + 64, qb * BQ);
            for (int j = 0; j < n_kv; ++j) {
                const int st = j & 1;
                mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
                mbar_expect_tx(&kv_full[st], 2 * kTile);
                uint8_t* kd = sm + FwdSmem::k + st * kTile;
                uint8_t* vd = sm + FwdSmem::v + st * kTile;
                tma_load_2d(kd, &tm_k, &kv_full[st], kvh * D, j * BKV);
                tma_load_2d(kd + kHalf, &tm_k, &kv_full[st], kvh * D + 64, j * BKV);
                tma_load_2d(vd, &tm_v, &kv_full[st], kvh * D, j * BKV);
                tma_load_2d(vd + kHalf, &tm_v, &kv_full[st], kvh * D + 64, j * BKV);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_s = umma_idesc_bf16(128, 128, false, false);
        constexpr uint32_t id_o = umma_idesc_bf16(128, 128, false, true);
        const uint32_t q_addr = smem_u32(sm + FwdSmem::q);
        const uint32_t p_addr = smem_u32(sm + FwdSmem::p);
        auto issue_s = [&](int j) {
            const int st = j & 1;
            mbar_wait(&kv_full[st], (j >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t k_addr = smem_u32(sm + FwdSmem::k + st * kTile);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    tc_mma_bf16(t_s0 + st * 128, desc_kmajor(q_addr, kk), desc_kmajor(k_addr, kk), id_s,
                                kk > 0);
                tc_commit(&s_full[st]);
            }
            __syncwarp();
        };
        mbar_wait(q_full, 0);
        issue_s(0);
        for (int j = 0; j < n_kv; ++j) {
            if (j + 1 < n_kv) issue_s(j + 1);
            mbar_wait(p_full, j & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t v_addr = smem_u32(sm + FwdSmem::v + (j & 1) * kTile);
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk)
                    tc_mma_bf16(t_o, desc_kmajor(p_addr, kk), desc_mnmajor(v_addr, kk), id_o,
                                (j | kk) != 0);
                tc_commit(&kv_empty[j & 1]);
                tc_commit(pv_done);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ softmax
        const int quad = warp & 3;
        const int r = quad * 32 + lane;                 // row within the tile
        const int qrow = qb * BQ + r;                   // query position
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        uint8_t* sp = sm + FwdSmem::p;
        float m_used = -INFINITY, l = 0.f;
        for (int j = 0; j < n_kv; ++j) {
            mbar_wait(&s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            float s[BKV];
#pragma unroll
            for (int c = 0; c < BKV / 32; ++c) {
                uint32_t rr[32];
                tmem_ld32(t_s0 + (j & 1) * 128 + lane_off + c * 32, rr);
                tmem_ld_wait();
#pragma unroll
                for (int t = 0; t < 32; ++t) s[c * 32 + t] = __uint_as_float(rr[t]) * p.scale_log2;
            }
            const bool diag = j == qb;
            float mx = -INFINITY;
#pragma unroll
            for (int t = 0; t < BKV; ++t) {
                const int key = j * BKV + t;
                if ((diag && key > qrow) || key >= p.T) s[t] = -INFINITY;
                mx = fmaxf(mx, s[t]);
            }
            // P smem and O are read by PV_{j-1}: wait for it before touching either.
            if (j > 0) mbar_wait(pv_done, (j - 1) & 1);
            tc_fence_after();
            if (mx > m_used + kRescaleThreshold || j == 0) {
                const float m_new = fmaxf(mx, m_used);
                if (j > 0) {
                    const float corr = fast_exp2(m_used - m_new);
                    l *= corr;
#pragma unroll 1
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t rr[32];
                        tmem_ld32(t_o + lane_off + c * 32, rr);
                        tmem_ld_wait();
#pragma unroll
                        for (int t = 0; t < 32; ++t) rr[t] = __float_as_uint(__uint_as_float(rr[t]) * corr);
                        tmem_st32(t_o + lane_off + c * 32, rr);
                    }
                    tmem_st_wait();
                }
                m_used = m_new;
            }
            float rs = 0.f;
#pragma unroll
            for (int c = 0; c < BKV / 8; ++c) {
                float pv[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    pv[t] = fast_exp2(s[c * 8 + t] - m_used);
                    rs += pv[t];
                }
                const int atom = c >> 3, cc = c & 7;
                *reinterpret_cast<uint4*>(sp + atom * kHalf + r * 128 + ((cc ^ (r & 7)) << 4)) = pack8(pv);
            }
            l += rs;
            fence_async_shared();  // generic-proxy smem writes -> visible to the MMA (async proxy)
            tc_fence_before();
            mbar_arrive(p_full);
        }
        mbar_wait(pv_done, (n_kv - 1) & 1);
        tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const bool ok = qrow < p.T;
        __nv_bfloat16* orow = p.o + static_cast<long long>(qrow) * p.ldo + h * D;
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
            uint32_t rr[32];
            tmem_ld32(t_o + lane_off + c * 32, rr);
            tmem_ld_wait();
            if (ok) {
#pragma unroll
                for (int t = 0; t < 32; t += 8) {
                    float f[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(rr[t + u]) * inv;
                    *reinterpret_cast<uint4*>(orow + c * 32 + t) = pack8(f);
                }
            }
        }
        if (ok) p.lse[static_cast<long long>(h) * p.T + qrow] = (m_used + log2f(l)) * (1.f / kLog2e);
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace

// Host launcher (dh_attn_fwd dispatches head_dim 128 here).
int attn_fwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv, void* o,
                long long ldo, float* lse, int T, int nq, int nkv, float scale, cudaStream_t s) {
    CUtensorMap mq, mk, mv;
    int rc = make_tma_2d(&mq, q, static_cast<long long>(nq) * D, T, ldq, 64, BQ);
    if (rc) return rc;
    rc = make_tma_2d(&mk, k, static_cast<long long>(nkv) * D, T, ldkv, 64, BKV);
    if (rc) return rc;
    rc = make_tma_2d(&mv, v, static_cast<long long>(nkv) * D, T, ldkv, 64, BKV);
    if (rc) return rc;
    static bool cfg = false;
    if (!cfg) {
        DH_CUDA_CHECK(cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           FwdSmem::total));
        cfg = true;
    }
    FwdParams prm{lse, static_cast<__nv_bfloat16*>(o), ldo, T, nq / nkv, scale * kLog2e};
    const dim3 grid((T + BQ - 1) / BQ, nq);
    attn_fwd_tc_kernel<<<grid, kThreads, FwdSmem::total, s>>>(mq, mk, mv, prm);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

}  // namespace dh
