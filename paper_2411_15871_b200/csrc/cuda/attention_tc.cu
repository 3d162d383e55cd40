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
    uint64_t* k_full = bars + 1;    // [2]  K ring: freed once S_j is computed
    uint64_t* k_empty = bars + 3;   // [2]
    uint64_t* s_full = bars + 5;    // [2]
    uint64_t* p_full = bars + 7;
    uint64_t* pv_done = bars + 8;
    uint64_t* v_full = bars + 9;    // [2]  V ring: freed once PV_j is accumulated
    uint64_t* v_empty = bars + 11;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

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
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
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
            // K runs up to two blocks ahead of V (it is released as soon as S_j is done)
            auto load_k = [&](int j) {
                const int st = j & 1;
                mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
                mbar_expect_tx(&k_full[st], kTile);
                uint8_t* kd = sm + FwdSmem::k + st * kTile;
                tma_load_2d(kd, &tm_k, &k_full[st], kvh * D, j * BKV);
                tma_load_2d(kd + kHalf, &tm_k, &k_full[st], kvh * D + 64, j * BKV);
            };
            auto load_v = [&](int j) {
                const int st = j & 1;
                mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
                mbar_expect_tx(&v_full[st], kTile);
                uint8_t* vd = sm + FwdSmem::v + st * kTile;
                tma_load_2d(vd, &tm_v, &v_full[st], kvh * D, j * BKV);
                tma_load_2d(vd + kHalf, &tm_v, &v_full[st], kvh * D + 64, j * BKV);
            };
            load_k(0);
            if (n_kv > 1) load_k(1);
            for (int j = 0; j < n_kv; ++j) {
                load_v(j);
                if (j + 2 < n_kv) load_k(j + 2);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_s = umma_idesc_bf16(128, 128, false, false);
        constexpr uint32_t id_o = umma_idesc_bf16(128, 128, false, true);
        const uint32_t q_addr = smem_u32(sm + FwdSmem::q);
        const uint32_t p_addr = smem_u32(sm + FwdSmem::p);
        auto issue_s = [&](int j) {
            const int st = j & 1;
            mbar_wait(&k_full[st], (j >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t k_addr = smem_u32(sm + FwdSmem::k + st * kTile);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    tc_mma_bf16(t_s0 + st * 128, desc_kmajor(q_addr, kk), desc_kmajor(k_addr, kk), id_s,
                                kk > 0);
                tc_commit(&s_full[st]);
                tc_commit(&k_empty[st]);
            }
            __syncwarp();
        };
        mbar_wait(q_full, 0);
        issue_s(0);
        for (int j = 0; j < n_kv; ++j) {
            if (j + 1 < n_kv) issue_s(j + 1);
            mbar_wait(p_full, j & 1);
            mbar_wait(&v_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t v_addr = smem_u32(sm + FwdSmem::v + (j & 1) * kTile);
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk)
                    tc_mma_bf16(t_o, desc_kmajor(p_addr, kk), desc_mnmajor(v_addr, kk), id_o,
                                (j | kk) != 0);
                tc_commit(&v_empty[j & 1]);
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
            // Lazy rescale. tcgen05.ld/st are warp-collective (.sync.aligned), so
            // the decision to touch O is made per warp (__any_sync); lanes that
            // do not need a new maximum rescale by exactly 1.
            const bool need = j == 0 || mx > m_used + kRescaleThreshold;
            const float m_new = need ? fmaxf(mx, m_used) : m_used;
            if (__any_sync(0xffffffffu, need && j > 0)) {
                const float corr = need ? fast_exp2(m_used - m_new) : 1.f;
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

// ===========================================================================
// Backward (attn_bwd node), two deterministic tcgen05 kernels.
//
// dK/dV kernel — one CTA per (128-key block, q head); inner q tiles of 64:
//   S^T  = K Q^T        M128 N64  K128   A=K (K-major)   B=Q (K-major)
//   dP^T = V dO^T       M128 N64  K128   A=V (K-major)   B=dO (K-major)
//   P^T = exp(scale S^T - lse_q), dS^T = P^T (dP^T - D_q)      (thread = key row)
//   dV  += P^T dO       M128 N128 K64    A=P^T (smem)    B=dO (MN-major)
//   dK  += dS^T Q       M128 N128 K64    A=dS^T (smem)   B=Q  (MN-major)
//   TMEM: S^T x2 (64) | dP^T x2 (64) | dV (128) | dK (128) = 512 columns.
// dQ kernel — one CTA per (128-query block, q head); inner key tiles of 64:
//   S = Q K^T, dP = dO V^T (M128 N64 K128), dS = P (dP - D)    (thread = query row)
//   dQ += dS K          M128 N128 K64    A=dS (smem)     B=K (MN-major)
//   TMEM: S x2 | dP x2 | dQ = 384 columns.
// No atomics: dQ is produced by its own pass and per-head dK/dV partials of a
// GQA group are reduced in head order by attn_bwd_group_reduce (attention.cu).
// ===========================================================================

namespace dh {
namespace {

constexpr int BT64 = 64;
constexpr int kTile64 = BT64 * D * 2;  // 16 KB: [2 d-halves][64 rows][128 B]
constexpr int kHalf64 = kTile64 / 2;   // 8 KB

struct KvSmem {
    static constexpr int k = 0;                      // 32 KB
    static constexpr int v = k + kTile;              // 32 KB
    static constexpr int q = v + kTile;              // 3 x 16 KB
    static constexpr int dout = q + 3 * kTile64;     // 3 x 16 KB
    static constexpr int pt = dout + 3 * kTile64;    // 2 x 16 KB  [128 keys][64 q]
    static constexpr int dst = pt + 2 * 16384;       // 2 x 16 KB
    static constexpr int vec = dst + 2 * 16384;      // per stage: lse[64], D[64] (raw)
    static constexpr int bars = vec + 3 * 128 * 4;
    static constexpr int total = bars + 256 + 1024;
};

struct BwdParams {
    const float* lse;
    const float* dvec;
    float* dk_part;
    float* dv_part;
    __nv_bfloat16* dk;
    __nv_bfloat16* dv;
    __nv_bfloat16* dq;
    long long lddkv, lddq;
    int T, group;
    float scale, scale_log2;
};

// K-major 64-row tile (one 64-wide K atom per half): k-step kk over d (0..7).
__device__ __forceinline__ uint64_t desc_k64(uint32_t base, int kk) {
    return umma_desc_sw128(base + (kk >> 2) * kHalf64 + (kk & 3) * 32, 16, 1024);
}
// MN-major 64-row tile used as B with N = d: k-step kk over rows (0..3).
__device__ __forceinline__ uint64_t desc_mn64(uint32_t base, int kk) {
    return umma_desc_sw128(base + kk * 2048, kHalf64, 1024);
}
// [128 rows][64 K] single-atom K-major tile (P^T, dS^T, dS): k-step kk (0..3).
__device__ __forceinline__ uint64_t desc_k1atom(uint32_t base, int kk) {
    return umma_desc_sw128(base + kk * 32, 16, 1024);
}

constexpr int kThreadsBwd = 320;  // producer, MMA, 8 elementwise warps (2 per TMEM quadrant)

__global__ void __launch_bounds__(kThreadsBwd, 1)
    attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                            const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                            const BwdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + KvSmem::bars);
    uint64_t* kv_full = bars + 0;
    uint64_t* q_full = bars + 1;   // [3] Q/dO ring
    uint64_t* q_empty = bars + 4;  // [3]
    uint64_t* s_full = bars + 7;   // [2] TMEM S^T/dP^T buffers
    uint64_t* p_full = bars + 9;
    uint64_t* mm_done = bars + 10;  // [2], one per P^T/dS^T buffer
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
    float* vec = reinterpret_cast<float*>(sm + KvSmem::vec);  // [stage][lse 64 | D 64]

    const int kb = gridDim.x - 1 - blockIdx.x;  // early key blocks see the most queries
    const int h = blockIdx.y;
    const int kvh = h / p.group;
    const int nq64 = (p.T + BT64 - 1) / BT64;
    const int i0 = (kb * D) / BT64;  // first q tile with a query >= the block's first key
    const int n_it = nq64 - i0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        mbar_init(kv_full, 1);
        for (int i = 0; i < 3; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
        mbar_init(p_full, 256);
        mbar_init(&mm_done[0], 1);
        mbar_init(&mm_done[1], 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t t_s = tmem, t_dp = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 384;
    const bool bulk_vec = (p.T % BT64) == 0;  // lse / D rows fetched by bulk copy

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(kv_full, 2 * kTile);
            tma_load_2d(sm + KvSmem::k, &tm_k, kv_full, kvh * D, kb * D);
            tma_load_2d(sm + KvSmem::k + kHalf, &tm_k, kv_full, kvh * D + 64, kb * D);
            tma_load_2d(sm + KvSmem::v, &tm_v, kv_full, kvh * D, kb * D);
            tma_load_2d(sm + KvSmem::v + kHalf, &tm_v, kv_full, kvh * D + 64, kb * D);
            for (int it = 0; it < n_it; ++it) {
                const int st = it % 3, qi = i0 + it;
                mbar_wait(&q_empty[st], ((it / 3) & 1) ^ 1);
                mbar_expect_tx(&q_full[st], 2 * kTile64 + (bulk_vec ? 512 : 0));
                if (bulk_vec) {
                    const long long off = static_cast<long long>(h) * p.T + qi * BT64;
                    bulk_load_1d(vec + st * 128, p.lse + off, 256, &q_full[st]);
                    bulk_load_1d(vec + st * 128 + 64, p.dvec + off, 256, &q_full[st]);
                }
                uint8_t* qd = sm + KvSmem::q + st * kTile64;
                uint8_t* od = sm + KvSmem::dout + st * kTile64;
                tma_load_2d(qd, &tm_q, &q_full[st], h * D, qi * BT64);
                tma_load_2d(qd + kHalf64, &tm_q, &q_full[st], h * D + 64, qi * BT64);
                tma_load_2d(od, &tm_do, &q_full[st], h * D, qi * BT64);
                tma_load_2d(od + kHalf64, &tm_do, &q_full[st], h * D + 64, qi * BT64);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_s = umma_idesc_bf16(128, 64, false, false);
        constexpr uint32_t id_g = umma_idesc_bf16(128, 128, false, true);
        const uint32_t k_addr = smem_u32(sm + KvSmem::k), v_addr = smem_u32(sm + KvSmem::v);
        const uint32_t pt_addr = smem_u32(sm + KvSmem::pt), ds_addr = smem_u32(sm + KvSmem::dst);
        auto issue_s = [&](int it) {
            const int qs = it % 3, sb = it & 1;  // smem ring stage, TMEM buffer
            mbar_wait(&q_full[qs], (it / 3) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t q_addr = smem_u32(sm + KvSmem::q + qs * kTile64);
                const uint32_t o_addr = smem_u32(sm + KvSmem::dout + qs * kTile64);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    tc_mma_bf16(t_s + sb * 64, desc_kmajor(k_addr, kk), desc_k64(q_addr, kk), id_s, kk > 0);
                    tc_mma_bf16(t_dp + sb * 64, desc_kmajor(v_addr, kk), desc_k64(o_addr, kk), id_s, kk > 0);
                }
                tc_commit(&s_full[sb]);
            }
            __syncwarp();
        };
        mbar_wait(kv_full, 0);
        if (n_it > 0) issue_s(0);
        for (int it = 0; it < n_it; ++it) {
            const int st = it & 1, qs = it % 3;
            if (it + 1 < n_it) issue_s(it + 1);
            mbar_wait(p_full, it & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t q_addr = smem_u32(sm + KvSmem::q + qs * kTile64);
                const uint32_t o_addr = smem_u32(sm + KvSmem::dout + qs * kTile64);
                const uint32_t pb = pt_addr + st * 16384, db = ds_addr + st * 16384;
#pragma unroll
                for (int kk = 0; kk < BT64 / 16; ++kk) {
                    tc_mma_bf16(t_dv, desc_k1atom(pb, kk), desc_mn64(o_addr, kk), id_g, (it | kk) != 0);
                    tc_mma_bf16(t_dk, desc_k1atom(db, kk), desc_mn64(q_addr, kk), id_g, (it | kk) != 0);
                }
                tc_commit(&q_empty[qs]);
                tc_commit(&mm_done[st]);
            }
            __syncwarp();
        }
    } else {
        // 8 warps: quadrant (TMEM lanes) = warp & 3, column half = (warp - 2) >> 2
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;
        const int r = quad * 32 + lane;  // key row within the block
        const int key = kb * D + r;
        const int t_sm = threadIdx.x - 64;  // 0..255 among the elementwise warps
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        uint8_t* spt = sm + KvSmem::pt;
        uint8_t* sds = sm + KvSmem::dst;
        const int key_hi = kb * D + D - 1;
        for (int it = 0; it < n_it; ++it) {
            const int st = it & 1, qi = i0 + it;
            if (!bulk_vec) {
                // ragged T: stage the vectors with plain loads (s_full implies q_full)
                named_barrier(1, 256);  // previous readers of this stage are done
                if (t_sm < BT64) {
                    const int q = qi * BT64 + t_sm;
                    vec[(it % 3) * 128 + t_sm] = q < p.T ? p.lse[static_cast<long long>(h) * p.T + q] : 0.f;
                    vec[(it % 3) * 128 + 64 + t_sm] = q < p.T ? p.dvec[static_cast<long long>(h) * p.T + q] : 0.f;
                }
                named_barrier(1, 256);
            }
            mbar_wait(&s_full[st], (it >> 1) & 1);
            tc_fence_after();
            uint32_t a[32], b[32];
            tmem_ld32(t_s + st * 64 + lane_off + half * 32, a);
            tmem_ld32(t_dp + st * 64 + lane_off + half * 32, b);
            tmem_ld_wait();
            // whole tile causal-visible and in range: no per-element masking
            const bool full_tile = qi * BT64 >= key_hi && qi * BT64 + BT64 <= p.T && key_hi < p.T;
            // This P^T / dS^T buffer was read by the dV/dK MMAs two iterations ago.
            if (it > 1) mbar_wait(&mm_done[st], ((it >> 1) - 1) & 1);
            const float* lv = vec + (it % 3) * 128 + half * 32;
            const float* dv_ = vec + (it % 3) * 128 + 64 + half * 32;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float pv[8], d8[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const int j = c * 8 + t;
                    float e = fast_exp2(__uint_as_float(a[j]) * p.scale_log2 - lv[j] * kLog2e);
                    if (!full_tile) {
                        const int q = qi * BT64 + half * 32 + j;
                        if (q < key || q >= p.T || key >= p.T) e = 0.f;
                    }
                    pv[t] = e;
                    d8[t] = e * (__uint_as_float(b[j]) - dv_[j]);
                }
                const int cc = half * 4 + c;
                const int off = st * 16384 + r * 128 + ((cc ^ (r & 7)) << 4);
                *reinterpret_cast<uint4*>(spt + off) = pack8(pv);
                *reinterpret_cast<uint4*>(sds + off) = pack8(d8);
            }
            fence_async_shared();
            tc_fence_before();
            mbar_arrive(p_full);
        }
        if (n_it > 0) mbar_wait(&mm_done[(n_it - 1) & 1], ((n_it - 1) >> 1) & 1);
        tc_fence_after();
        const bool ok = key < p.T;
#pragma unroll 1
        for (int c = half * 2; c < half * 2 + 2; ++c) {
            uint32_t ka[32], va[32];
            tmem_ld32(t_dk + lane_off + c * 32, ka);
            tmem_ld32(t_dv + lane_off + c * 32, va);
            tmem_ld_wait();
            if (!ok) continue;
            if (p.group == 1) {
                __nv_bfloat16* kr = p.dk + static_cast<long long>(key) * p.lddkv + kvh * D + c * 32;
                __nv_bfloat16* vr = p.dv + static_cast<long long>(key) * p.lddkv + kvh * D + c * 32;
#pragma unroll
                for (int t = 0; t < 32; t += 8) {
                    float fk[8], fv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        fk[u] = n_it > 0 ? __uint_as_float(ka[t + u]) * p.scale : 0.f;
                        fv[u] = n_it > 0 ? __uint_as_float(va[t + u]) : 0.f;
                    }
                    *reinterpret_cast<uint4*>(kr + t) = pack8(fk);
                    *reinterpret_cast<uint4*>(vr + t) = pack8(fv);
                }
            } else {
                float* kr = p.dk_part + (static_cast<long long>(h) * p.T + key) * D + c * 32;
                float* vr = p.dv_part + (static_cast<long long>(h) * p.T + key) * D + c * 32;
#pragma unroll
                for (int t = 0; t < 32; t += 4) {
                    *reinterpret_cast<float4*>(kr + t) =
                        make_float4(__uint_as_float(ka[t]) * p.scale, __uint_as_float(ka[t + 1]) * p.scale,
                                    __uint_as_float(ka[t + 2]) * p.scale, __uint_as_float(ka[t + 3]) * p.scale);
                    *reinterpret_cast<float4*>(vr + t) =
                        make_float4(__uint_as_float(va[t]), __uint_as_float(va[t + 1]),
                                    __uint_as_float(va[t + 2]), __uint_as_float(va[t + 3]));
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

struct DqSmem {
    static constexpr int q = 0;                      // 32 KB
    static constexpr int dout = q + kTile;           // 32 KB
    static constexpr int k = dout + kTile;           // 3 x 16 KB
    static constexpr int v = k + 3 * kTile64;        // 3 x 16 KB
    static constexpr int ds = v + 3 * kTile64;       // 2 x 16 KB [128 q][64 keys]
    static constexpr int bars = ds + 2 * 16384;
    static constexpr int total = bars + 256 + 1024;
};

__global__ void __launch_bounds__(kThreadsBwd, 1)
    attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                          const BwdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + DqSmem::bars);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;   // [3] K/V ring
    uint64_t* kv_empty = bars + 4;  // [3]
    uint64_t* s_full = bars + 7;    // [2]
    uint64_t* p_full = bars + 9;
    uint64_t* mm_done = bars + 10;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

    const int qb = gridDim.x - 1 - blockIdx.x;
    const int h = blockIdx.y;
    const int kvh = h / p.group;
    const int n_it = (qb * D + D) / BT64;  // key tiles 0 .. covering the block's last query
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        mbar_init(q_full, 1);
        for (int i = 0; i < 3; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
        mbar_init(p_full, 256);
        mbar_init(&mm_done[0], 1);
        mbar_init(&mm_done[1], 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t t_s = tmem, t_dp = tmem + 128, t_dq = tmem + 256;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(q_full, 2 * kTile);
            tma_load_2d(sm + DqSmem::q, &tm_q, q_full, h * D, qb * D);
            tma_load_2d(sm + DqSmem::q + kHalf, &tm_q, q_full, h * D + 64, qb * D);
            tma_load_2d(sm + DqSmem::dout, &tm_do, q_full, h * D, qb * D);
            tma_load_2d(sm + DqSmem::dout + kHalf, &tm_do, q_full, h * D + 64, qb * D);
            for (int it = 0; it < n_it; ++it) {
                const int st = it % 3;
                mbar_wait(&kv_empty[st], ((it / 3) & 1) ^ 1);
                mbar_expect_tx(&kv_full[st], 2 * kTile64);
                uint8_t* kd = sm + DqSmem::k + st * kTile64;
                uint8_t* vd = sm + DqSmem::v + st * kTile64;
                tma_load_2d(kd, &tm_k, &kv_full[st], kvh * D, it * BT64);
                tma_load_2d(kd + kHalf64, &tm_k, &kv_full[st], kvh * D + 64, it * BT64);
                tma_load_2d(vd, &tm_v, &kv_full[st], kvh * D, it * BT64);
                tma_load_2d(vd + kHalf64, &tm_v, &kv_full[st], kvh * D + 64, it * BT64);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_s = umma_idesc_bf16(128, 64, false, false);
        constexpr uint32_t id_g = umma_idesc_bf16(128, 128, false, true);
        const uint32_t q_addr = smem_u32(sm + DqSmem::q), o_addr = smem_u32(sm + DqSmem::dout);
        const uint32_t ds_addr = smem_u32(sm + DqSmem::ds);
        auto issue_s = [&](int it) {
            const int ks = it % 3, sb = it & 1;
            mbar_wait(&kv_full[ks], (it / 3) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t k_addr = smem_u32(sm + DqSmem::k + ks * kTile64);
                const uint32_t v_addr = smem_u32(sm + DqSmem::v + ks * kTile64);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    tc_mma_bf16(t_s + sb * 64, desc_kmajor(q_addr, kk), desc_k64(k_addr, kk), id_s, kk > 0);
                    tc_mma_bf16(t_dp + sb * 64, desc_kmajor(o_addr, kk), desc_k64(v_addr, kk), id_s, kk > 0);
                }
                tc_commit(&s_full[sb]);
            }
            __syncwarp();
        };
        mbar_wait(q_full, 0);
        issue_s(0);
        for (int it = 0; it < n_it; ++it) {
            const int st = it & 1, ks = it % 3;
            if (it + 1 < n_it) issue_s(it + 1);
            mbar_wait(p_full, it & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t k_addr = smem_u32(sm + DqSmem::k + ks * kTile64);
#pragma unroll
                for (int kk = 0; kk < BT64 / 16; ++kk)
                    tc_mma_bf16(t_dq, desc_k1atom(ds_addr + st * 16384, kk), desc_mn64(k_addr, kk), id_g,
                                (it | kk) != 0);
                tc_commit(&kv_empty[ks]);
                tc_commit(&mm_done[st]);
            }
            __syncwarp();
        }
    } else {
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;
        const int r = quad * 32 + lane;
        const int qrow = qb * D + r;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const int qc = min(qrow, p.T - 1);
        const float lse2 = p.lse[static_cast<long long>(h) * p.T + qc] * kLog2e;
        const float dd = p.dvec[static_cast<long long>(h) * p.T + qc];
        uint8_t* sds = sm + DqSmem::ds;
        for (int it = 0; it < n_it; ++it) {
            const int st = it & 1;
            mbar_wait(&s_full[st], (it >> 1) & 1);
            tc_fence_after();
            uint32_t a[32], b[32];
            tmem_ld32(t_s + st * 64 + lane_off + half * 32, a);
            tmem_ld32(t_dp + st * 64 + lane_off + half * 32, b);
            tmem_ld_wait();
            const bool full_tile = it * BT64 + BT64 - 1 <= qb * D && it * BT64 + BT64 <= p.T && qb * D + D <= p.T;
            if (it > 1) mbar_wait(&mm_done[st], ((it >> 1) - 1) & 1);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float d8[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const int j = c * 8 + t;
                    float e = fast_exp2(__uint_as_float(a[j]) * p.scale_log2 - lse2);
                    if (!full_tile) {
                        const int key = it * BT64 + half * 32 + j;
                        if (key > qrow || key >= p.T) e = 0.f;
                    }
                    d8[t] = e * (__uint_as_float(b[j]) - dd);
                }
                const int cc = half * 4 + c;
                *reinterpret_cast<uint4*>(sds + st * 16384 + r * 128 + ((cc ^ (r & 7)) << 4)) = pack8(d8);
            }
            fence_async_shared();
            tc_fence_before();
            mbar_arrive(p_full);
        }
        mbar_wait(&mm_done[(n_it - 1) & 1], ((n_it - 1) >> 1) & 1);
        tc_fence_after();
        const bool ok = qrow < p.T;
        __nv_bfloat16* row = p.dq + static_cast<long long>(qrow) * p.lddq + h * D;
#pragma unroll 1
        for (int c = half * 2; c < half * 2 + 2; ++c) {
            uint32_t a[32];
            tmem_ld32(t_dq + lane_off + c * 32, a);
            tmem_ld_wait();
            if (!ok) continue;
#pragma unroll
            for (int t = 0; t < 32; t += 8) {
                float f[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(a[t + u]) * p.scale;
                *reinterpret_cast<uint4*>(row + c * 32 + t) = pack8(f);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace

// Host launcher for the two tcgen05 backward kernels (dvec must already hold
// D_i = rowsum(dO * O)); dk_part / dv_part are used only when group > 1.
int attn_bwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                const void* dout, long long ldo, const float* lse, const float* dvec, float* dk_part,
                float* dv_part, void* dq, void* dk, void* dv, long long lddq, long long lddkv, int T,
                int nq, int nkv, float scale, cudaStream_t s) {
    CUtensorMap mk, mv, mq64, mdo64, mq, mdo, mk64, mv64;
    const long long qcols = static_cast<long long>(nq) * D, kvcols = static_cast<long long>(nkv) * D;
    int rc = make_tma_2d(&mk, k, kvcols, T, ldkv, 64, 128);
    if (!rc) rc = make_tma_2d(&mv, v, kvcols, T, ldkv, 64, 128);
    if (!rc) rc = make_tma_2d(&mq64, q, qcols, T, ldq, 64, 64);
    if (!rc) rc = make_tma_2d(&mdo64, dout, qcols, T, ldo, 64, 64);
    if (!rc) rc = make_tma_2d(&mq, q, qcols, T, ldq, 64, 128);
    if (!rc) rc = make_tma_2d(&mdo, dout, qcols, T, ldo, 64, 128);
    if (!rc) rc = make_tma_2d(&mk64, k, kvcols, T, ldkv, 64, 64);
    if (!rc) rc = make_tma_2d(&mv64, v, kvcols, T, ldkv, 64, 64);
    if (rc) return rc;
    static bool cfg = false;
    if (!cfg) {
        DH_CUDA_CHECK(cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, KvSmem::total));
        DH_CUDA_CHECK(cudaFuncSetAttribute(attn_bwd_dq_tc_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, DqSmem::total));
        cfg = true;
    }
    BwdParams prm{lse, dvec, dk_part, dv_part, static_cast<__nv_bfloat16*>(dk),
                  static_cast<__nv_bfloat16*>(dv), static_cast<__nv_bfloat16*>(dq), lddkv, lddq, T,
                  nq / nkv, scale, scale * kLog2e};
    const int nb = (T + D - 1) / D;
    attn_bwd_dkdv_tc_kernel<<<dim3(nb, nq), kThreadsBwd, KvSmem::total, s>>>(mk, mv, mq64, mdo64, prm);
    DH_CUDA_CHECK(cudaGetLastError());
    attn_bwd_dq_tc_kernel<<<dim3(nb, nq), kThreadsBwd, DqSmem::total, s>>>(mq, mdo, mk64, mv64, prm);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

}  // namespace dh
