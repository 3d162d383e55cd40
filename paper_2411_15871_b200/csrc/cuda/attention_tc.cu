// Causal GQA flash attention on tcgen05 / TMEM / TMA (head_dim 64 or 128) —
// the attn node (forward) and attn_bwd (backward). Every kernel is a template
// on the head dimension D: a 128-row tile of D columns is D/64 swizzle atoms
// ("d-halves") of 64 bf16 each, so D = 64 is one atom and D = 128 two.
//
// One CTA per work item = (pair of 128-query tiles of one q head[, KV chunk]);
// KV blocks of 128 keys, causal blocks only, items dispatched heaviest first
// across heads. The two query tiles ping-pong on the tensor core: while the
// softmax warps of one tile turn S into P, the MMA warp runs the other tile's
// PV and next QK^T, so the tensor pipe is not idle during the softmax.
// When the grid is too small to balance (few heads per GPU at high TP: the
// longest causal row is the critical path), long rows are split into KV
// chunks chosen by an LPT makespan model on the host; each chunk writes an
// unnormalised fp32 partial (O, max, sum) and attn_fwd_combine merges them.
//   warp 0       TMA producer: Q tiles once, K_j / V_j through a 5-slot ring
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5   softmax of tile 0, warps 6..9 softmax of tile 1
//                (thread = query row = its TMEM lane)
// TMEM (512 cols): S0 | S1 | O0 | O1 (128 columns each).
//   S_t  = Q_t K_j^T         M128 N128 K128, A=Q (smem, K-major), B=K (smem, K-major)
//   P_t  = exp2(S_t ...)     bf16, written back over the first 64 columns of S_t
//   O_t += P_t V_j           M128 N128 K128, A=P (TMEM), B=V (smem, MN-major)
// The same smem tile of K/V rows serves as K-major B for QK^T and as MN-major
// B for PV (only the descriptor differs). P never touches shared memory, which
// keeps the SS-mode QK^T below the shared-memory bandwidth limit. Online
// softmax uses lazy rescaling: O (in TMEM) is only rescaled when a row maximum
// grows by more than 2^8; P values are bounded by 2^8 in between.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>
#include <utility>
#include <vector>

#include "common.cuh"
#include "dh_capi.h"

#ifdef DH_ATTN_TRACE
__device__ long long g_attn_trace[1 << 14];
extern "C" int dh_attn_trace_read(long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(long long) * n) == cudaSuccess ? 0 : 1;
}
#define ATR(idx) do { if (blockIdx.x == DH_ATTN_TRACE) g_attn_trace[(idx)] = clock64(); } while (0)
#else
#define ATR(idx) do { } while (0)
#endif
#ifdef DH_ATTN_BLKTRACE
// per-block (start ns, end ns, SM id) of the last backward launch (tools/attn_blocks.py)
__device__ unsigned long long g_attn_blk[8192 * 3];
extern "C" int dh_attn_blk_read(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_attn_blk, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
__device__ __forceinline__ void blk_stamp(int i) {
    if (threadIdx.x == 0 && blockIdx.x < 8192) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_attn_blk[blockIdx.x * 3 + i] = t;
        if (i == 0) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            g_attn_blk[blockIdx.x * 3 + 2] = sm;
        }
    }
}
#define BLK(i) blk_stamp(i)
// forward phases per block (globaltimer ns): [0] prologue done, [1] Q and K_0
// landed (MMA warp), [2] first S_0 ready (softmax tile 0), [3] tile 0's O done,
// [4] tile 0's epilogue stores issued
__device__ unsigned long long g_attn_ph[8192 * 8];
extern "C" int dh_attn_phase_read(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_attn_ph, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#define PH(i, cond)                                                        \
    do {                                                                   \
        if ((cond) && blockIdx.x < 8192) {                                 \
            unsigned long long t_;                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));         \
            g_attn_ph[blockIdx.x * 8 + (i)] = t_;                          \
        }                                                                  \
    } while (0)
#else
#define BLK(i) do { } while (0)
#define PH(i, cond) do { } while (0)
#endif

namespace dh {
namespace {

constexpr int BQ = 128;
constexpr int BKV = 128;
constexpr int kThreads = 320;
// a 128-row tile: [D/64 d-halves][128 rows][128 B] (32 KB at D = 128)
template <int D>
constexpr int tile_bytes() { return BQ * D * 2; }
constexpr int kHalf = BQ * 64 * 2;      // 16 KB: one d-half of a 128-row tile
constexpr int kRing = 5;                // K/V tiles in flight: ring index 2j = K_j, 2j+1 = V_j
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.f;  // log2 units
#ifndef DH_ATTN_POLY
#define DH_ATTN_POLY 1
#endif
// quarters of the forward's / backward's exponentials on the FMA pipe (0..3)
#ifndef DH_ATTN_FWD_POLY_Q
#define DH_ATTN_FWD_POLY_Q 1
#endif
#ifndef DH_ATTN_BWD_POLY_Q
#define DH_ATTN_BWD_POLY_Q 1
#endif

template <int D>
struct FwdSmem {
    static constexpr int kTile = tile_bytes<D>();
    // offsets from the 1024-aligned base
    static constexpr int q = 0;                  // two query tiles
    static constexpr int kv = q + 2 * kTile;     // kRing slots
    static constexpr int bars = kv + kRing * kTile;
    static constexpr int total = bars + 256 + 1024;
};
static_assert(FwdSmem<128>::total <= 232448, "forward smem exceeds the sm_100 limit");

struct FwdParams {
    float* lse;
    __nv_bfloat16* o;
    long long ldo;
    int T;         // query rows (this rank's)
    int group;
    float scale_log2;
    int nq;        // q heads (item index = rank * nq + head)
    int nkb;       // 128-key blocks of the keys (T_kv)
    int npairs;    // query-tile pairs
    int chunk;     // KV blocks per chunk (even); 0 = no split
    int maxc;      // chunks of the longest row
    float* part;   // split partials: O [h][qb][c][d][row], then (m, l) [h][qb][c][row][2]
    int T_kv;      // key rows
    int qo;        // query offset in 128-blocks (context parallelism: the rank's first
                   // query sits at global position qo * 128; even, so chunks stay even)
};

constexpr int kMaxItems = 1024;  // split schedule entries per head (kernel parameter)
struct FwdSched {
    uint32_t item[kMaxItems];  // (pair << 16) | chunk, heaviest first
};

// (2^x0, 2^x1) for x <= 0 on the FMA pipe, packed fp32x2: x = n + f
// (n = round(x), |f| <= 1/2), 2^f by a degree-3 polynomial (max relative
// error 1.2e-4, below bf16's 2^-9 rounding of P), 2^n added to the exponent
// bits. x is clamped at -125, so masked (-inf) scores give 2^-125, which
// vanishes against any unmasked term.
__device__ __forceinline__ uint64_t exp2_fma2(float x0, float x1) {
    const uint64_t x = f2_pack(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
    const uint64_t t = fadd2(x, f2_pack(12582912.f, 12582912.f));  // 1.5 * 2^23: round to an integer
    const uint64_t fr = ffma2(fadd2(t, f2_pack(-12582912.f, -12582912.f)), f2_pack(-1.f, -1.f), x);
    uint64_t q = ffma2(f2_pack(0.05459283f, 0.05459283f), fr, f2_pack(0.24221838f, 0.24221838f));
    q = ffma2(q, fr, f2_pack(0.69336867f, 0.69336867f));
    q = ffma2(q, fr, f2_pack(1.f, 1.f));
    float q0, q1, t0, t1;
    f2_unpack(q, q0, q1);
    f2_unpack(t, t0, t1);
    return f2_pack(__int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23)),
                   __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23)));
}

// K-major operand, 2 swizzle atoms along K (d or keys): k-step kk of 16.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int kk) {
    return umma_desc_sw128(base + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
}
// MN-major operand (V as B with N = d): k-step kk of 16 keys.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int kk) {
    return umma_desc_sw128(base + kk * 2048, kHalf, 1024);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const FwdParams p,
                       const __grid_constant__ FwdSched sched) {
    using FwdSmem = dh::FwdSmem<D>;
    constexpr int kTile = FwdSmem::kTile;
    BLK(0);
    extern __shared__ uint8_t smem_raw[];
    // offset arithmetic on the __shared__ array keeps the pointer in the shared
    // space (plain loads compile to LDS rather than generic LD)
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + FwdSmem::bars);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;            // [kRing]
    uint64_t* kv_empty = bars + 1 + kRing;   // [kRing]
    uint64_t* s_full = bars + 1 + 2 * kRing;  // [2] per tile: S_t(j) computed (and PV_t(j-1) done)
    uint64_t* p_full = s_full + 2;           // [2] per tile: P_t(j) in TMEM
    uint64_t* o_done = s_full + 4;           // [2] per tile: last PV done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 6);

    const int rank = blockIdx.x / p.nq;
    const int h = blockIdx.x % p.nq;
    int qp, ch = 0, kv0 = 0, kvend;
    if (p.chunk) {
        const uint32_t e = sched.item[rank];
        qp = static_cast<int>(e >> 16);
        ch = static_cast<int>(e & 0xffffu);
        kv0 = ch * p.chunk;
        kvend = min(kv0 + p.chunk, p.qo + 2 * qp + 2);
    } else {
        qp = p.npairs - 1 - rank;
        kvend = p.qo + 2 * qp + 2;  // causal, BQ == BKV
    }
    kvend = min(kvend, p.nkb);
    const bool split = p.chunk && p.qo + 2 * qp + 2 > p.chunk;
    const int kvh = h / p.group;
    const int n = kvend - kv0;                              // blocks of tile 1
    const int n0 = min(kvend, p.qo + 2 * qp + 1) - kv0;     // blocks of tile 0 (n or n - 1; >= 1: chunks are even)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        mbar_init(q_full, 1);
        for (int i = 0; i < kRing; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&p_full[t], 128);
            mbar_init(&o_done[t], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t t_s = tmem, t_o = tmem + 256;  // S_t at t_s + 128 t, O_t at t_o + 128 t
    PH(0, threadIdx.x == 0);

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(q_full, 2 * kTile);
            for (int t = 0; t < 2; ++t) {
                uint8_t* qd = sm + FwdSmem::q + t * kTile;
#pragma unroll
                for (int hh = 0; hh < D / 64; ++hh)
                    tma_load_2d(qd + hh * kHalf, &tm_q, q_full, h * D + 64 * hh, (2 * qp + t) * BQ);
            }
            for (int idx = 0; idx < 2 * n; ++idx) {
                const int slot = idx % kRing;
                mbar_wait(&kv_empty[slot], ((idx / kRing) & 1) ^ 1);
                mbar_expect_tx(&kv_full[slot], kTile);
                uint8_t* dst = sm + FwdSmem::kv + slot * kTile;
                const CUtensorMap* map = (idx & 1) ? &tm_v : &tm_k;
                const int row = (kv0 + (idx >> 1)) * BKV;
#pragma unroll
                for (int hh = 0; hh < D / 64; ++hh)
                    tma_load_2d(dst + hh * kHalf, map, &kv_full[slot], kvh * D + 64 * hh, row);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_s = umma_idesc_bf16(128, 128, false, false);
        constexpr uint32_t id_o = umma_idesc_bf16(128, D, false, true);
        const uint32_t q_addr = smem_u32(sm + FwdSmem::q);
        const uint32_t kv_addr = smem_u32(sm + FwdSmem::kv);
        auto wait_kv = [&](int idx) {
            mbar_wait(&kv_full[idx % kRing], (idx / kRing) & 1);
            tc_fence_after();
        };
        auto issue_s = [&](int t, int j) {  // S_t = Q_t K_j^T
            if (elect_one()) {
                const uint32_t k_addr = kv_addr + ((2 * j) % kRing) * kTile;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    tc_mma_bf16(t_s + t * 128, desc_kmajor(q_addr + t * kTile, kk), desc_kmajor(k_addr, kk), id_s,
                                kk > 0);
                tc_commit(&s_full[t]);
            }
            __syncwarp();
        };
        auto release = [&](int idx) {
            if (elect_one()) tc_commit(&kv_empty[idx % kRing]);
            __syncwarp();
        };
        mbar_wait(q_full, 0);
        wait_kv(0);
        PH(1, lane == 0);
        issue_s(0, 0);
        issue_s(1, 0);
        release(0);
        for (int j = 0; j < n; ++j) {
            wait_kv(2 * j + 1);  // V_j
            const uint32_t v_addr = kv_addr + ((2 * j + 1) % kRing) * kTile;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int nt = t ? n : n0;
                if (j >= nt) continue;
                mbar_wait(&p_full[t], j & 1);
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < BKV / 16; ++kk)
                        tc_mma_bf16_ts(t_o + t * 128, t_s + t * 128 + kk * 8, desc_mnmajor(v_addr, kk), id_o,
                                       (j | kk) != 0);
                    if (j + 1 >= nt) tc_commit(&o_done[t]);
                }
                __syncwarp();
                if (t == 1) release(2 * j + 1);  // tile 1 is the last reader of V_j
                if (j + 1 < nt) {
                    wait_kv(2 * j + 2);  // K_{j+1}
                    issue_s(t, j + 1);
                    if (t == 1) release(2 * j + 2);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ softmax
        const int t = (warp - 2) >> 2;
        const int quad = warp & 3;
        const int r = quad * 32 + lane;                 // row within the tile
        const int qb = 2 * qp + t;                      // query block of this tile
        const int qrow = qb * BQ + r;                   // query row (this rank's)
        const int qpos = (p.qo + qb) * BQ + r;          // its global position (causal mask)
        const int nt = t ? n : n0;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t ts = t_s + t * 128 + lane_off, to = t_o + t * 128 + lane_off;
        float m_used = -INFINITY, l = 0.f;
        for (int j = 0; j < nt; ++j) {
            mbar_wait(&s_full[t], j & 1);
            tc_fence_after();
            PH(2, j == 0 && t == 0 && r == 0);
            // all four 32-column loads in flight before one wait
            uint32_t sr[BKV];
#pragma unroll
            for (int c = 0; c < BKV / 32; ++c) tmem_ld32(ts + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + c * 32));
            tmem_ld_wait();
            const int kb = kv0 + j;
            const bool masked = kb == p.qo + qb || (kb + 1) * BKV > p.T_kv;
            auto apply_mask = [&](int c0, int c1) {
#pragma unroll
                for (int u = c0; u < c1; ++u) {
                    const int key = kb * BKV + u;
                    if (key > qpos || key >= p.T_kv) sr[u] = __float_as_uint(-INFINITY);
                }
            };
            if (masked) apply_mask(0, BKV);
            // row max as 8 independent chains (a single 128-long dependent
            // FMNMX chain was the softmax critical path)
            float m8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) m8[u] = __uint_as_float(sr[u]);
#pragma unroll
            for (int u = 8; u < BKV; u += 16)
#pragma unroll
                for (int w = 0; w < 8; ++w)
                    m8[w] = fmax3(m8[w], __uint_as_float(sr[u + w]), __uint_as_float(sr[u + 8 + w < BKV ? u + 8 + w : u + w]));
            const float mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7])) *
                             p.scale_log2;
            // Lazy rescale. S_t(j) was issued after PV_t(j-1), so s_full also
            // means O_t is quiescent. tcgen05.ld/st are warp-collective, so the
            // decision to touch O is made per warp (__any_sync); lanes that do
            // not need a new maximum rescale by exactly 1.
            const bool need = j == 0 || mx > m_used + kRescaleThreshold;
            const float m_new = need ? fmaxf(mx, m_used) : m_used;
            if (__any_sync(0xffffffffu, need && j > 0)) {
                const float corr = need ? fast_exp2(m_used - m_new) : 1.f;
                l *= corr;
#pragma unroll 1
                for (int c = 0; c < D / 32; ++c) {
                    uint32_t rr[32];
                    tmem_ld32(to + c * 32, rr);
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 32; ++u) rr[u] = __float_as_uint(__uint_as_float(rr[u]) * corr);
                    tmem_st32(to + c * 32, rr);
                }
            }
            m_used = m_new;
            const uint64_t neg_m = f2_pack(-m_used, -m_used), sc2 = f2_pack(p.scale_log2, p.scale_log2);
            uint64_t r4[4] = {0, 0, 0, 0};  // packed row-sum partials
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                if (c == 1) {
                    // columns 64..127 are reloaded rather than kept live across
                    // the first half: the register budget is 168 at 10 warps
                    tmem_ld32(ts + 64, *reinterpret_cast<uint32_t(*)[32]>(sr + 64));
                    tmem_ld32(ts + 96, *reinterpret_cast<uint32_t(*)[32]>(sr + 96));
                    tmem_ld_wait();
                    if (masked) apply_mask(64, BKV);
                }
                uint32_t pk[32];
#pragma unroll
                for (int u = 0; u < 32; ++u) {
                    const int e = c * 64 + 2 * u;
                    const uint64_t x = ffma2(f2_pack(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])), sc2, neg_m);
                    // a quarter of the exponentials run on the FMA pipe: both
                    // softmax tiles together would otherwise saturate the MUFU
                    uint64_t pp;
                    if (DH_ATTN_POLY && (u & 3) >= 4 - DH_ATTN_FWD_POLY_Q) {
                        float x0, x1;
                        f2_unpack(x, x0, x1);
                        pp = exp2_fma2(x0, x1);
                    } else {
                        float x0, x1;
                        f2_unpack(x, x0, x1);
                        pp = f2_pack(fast_exp2(x0), fast_exp2(x1));
                    }
                    r4[u & 3] = fadd2(r4[u & 3], pp);
                    float p0, p1;
                    f2_unpack(pp, p0, p1);
                    pk[u] = pack2(p0, p1);
                }
                tmem_st32(ts + c * 32, pk);  // P over S columns [0, 64)
            }
            float ra, rb, rc, rd;
            f2_unpack(fadd2(fadd2(r4[0], r4[1]), fadd2(r4[2], r4[3])), ra, rb);
            (void)rc;
            (void)rd;
            const float rs = ra + rb;
            l += rs;
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[t]);
        }
        mbar_wait(&o_done[t], 0);
        tc_fence_after();
        PH(3, t == 0 && r == 0);
        if (split) {
            // unnormalised partial, [d][row] so a warp's stores are coalesced
            const long long slot = (static_cast<long long>(h) * (2 * p.npairs) + qb) * p.maxc + ch;
            float* po = p.part + slot * (BQ * D) + r;
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
                uint32_t rr[32];
                tmem_ld32(to + c * 32, rr);
                tmem_ld_wait();
#pragma unroll
                for (int u = 0; u < 32; ++u) po[(c * 32 + u) * BQ] = __uint_as_float(rr[u]);
            }
            float* pml = p.part + static_cast<long long>(p.nq) * (2 * p.npairs) * p.maxc * (BQ * D) +
                         slot * (2 * BQ);
            *reinterpret_cast<float2*>(pml + 2 * r) = make_float2(m_used, l);
            PH(4, t == 0 && r == 0);
        } else {
            const float inv = l > 0.f ? 1.f / l : 0.f;
            const bool ok = qrow < p.T;
            __nv_bfloat16* orow = p.o + static_cast<long long>(qrow) * p.ldo + h * D;
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
                uint32_t rr[32];
                tmem_ld32(to + c * 32, rr);
                tmem_ld_wait();
                if (ok) {
#pragma unroll
                    for (int u = 0; u < 32; u += 8) {
                        float f[8];
#pragma unroll
                        for (int w = 0; w < 8; ++w) f[w] = __uint_as_float(rr[u + w]) * inv;
                        *reinterpret_cast<uint4*>(orow + c * 32 + u) = pack8(f);
                    }
                }
            }
            if (ok) p.lse[static_cast<long long>(h) * p.T + qrow] = (m_used + log2f(l)) * (1.f / kLog2e);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
    BLK(1);
}

// Merge the KV-chunk partials of every split row: O = sum_c 2^(m_c-M) O_c / L,
// L = sum_c 2^(m_c-M) l_c, lse = (M + log2 L) ln 2. Chunks are merged in chunk
// order, so the result is deterministic. Block = (query block, head, 16-column
// slice of d); thread = (row, 8 columns): partial loads are coalesced along
// rows ([d][row] layout). Blocks of unsplit rows (fewer than 2 chunks) exit.
template <int D>
constexpr int combine_slices() { return D / 16; }
// MAXC >= the row's chunk count: every load is issued unconditionally (chunk
// indices clamped, surplus chunks weighted 0), so a thread has all of its
// MAXC x 8 partial loads in flight at once instead of one dependent L2 round
// trip per chunk and column.
template <int MAXC, int D>
__global__ void __launch_bounds__(256) attn_fwd_combine_kernel(const FwdParams p) {
    const int h = blockIdx.y;
    const int qb = blockIdx.x;
    const int nblk = min(p.qo + 2 * (qb >> 1) + 2, p.nkb);
    const int nc = (nblk + p.chunk - 1) / p.chunk;
    const int r = threadIdx.x & (BQ - 1);
    const int d0 = blockIdx.z * 16 + (threadIdx.x >> 7) * 8;
    const int qrow = qb * BQ + r;
    if (qrow >= p.T || nc < 2) return;
    const long long slot0 = (static_cast<long long>(h) * (2 * p.npairs) + qb) * p.maxc;
    const float* pml = p.part + static_cast<long long>(p.nq) * (2 * p.npairs) * p.maxc * (BQ * D);
    float2 ml[MAXC];
    float pv[MAXC][8];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        const long long sc = slot0 + min(c, nc - 1);
        ml[c] = *reinterpret_cast<const float2*>(pml + sc * (2 * BQ) + 2 * r);
        const float* po = p.part + sc * (BQ * D) + r;
#pragma unroll
        for (int u = 0; u < 8; ++u) pv[c][u] = po[(d0 + u) * BQ];
    }
    float M = -INFINITY;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) M = c < nc ? fmaxf(M, ml[c].x) : M;
    float L = 0.f, f[8] = {};
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        if (c < nc) {  // chunk order: deterministic
            const float w = exp2f(ml[c].x - M);
            L += w * ml[c].y;
#pragma unroll
            for (int u = 0; u < 8; ++u) f[u] += w * pv[c][u];
        }
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) f[u] *= inv;
    *reinterpret_cast<uint4*>(p.o + static_cast<long long>(qrow) * p.ldo + h * D + d0) = pack8(f);
    if (blockIdx.z == 0 && threadIdx.x < BQ)
        p.lse[static_cast<long long>(h) * p.T + qrow] = (M + log2f(L)) * (1.f / kLog2e);
}

// Split plan for a causal forward: LPT makespan over the SMs of the item costs
// in KV-block units of a tile pair (blocks + fixed per-item cost + partial
// write/merge for split items). Chunks are even so that both tiles of a pair
// always have work in every chunk.
struct FwdSplit {
    int chunk = 0, maxc = 1, items = 0;
    FwdSched sched;
};

// KV blocks a query-tile pair reads: causal up to its second tile's diagonal
int pair_blocks(int qp, int qo, int nkb) { return std::min(qo + 2 * qp + 2, nkb); }

double fwd_makespan(int nq, int npairs, int qo, int nkb, int chunk, int sms,
                    std::vector<std::pair<float, uint32_t>>* out) {
    std::vector<std::pair<float, uint32_t>> it;
    for (int qp = 0; qp < npairs; ++qp) {
        const int nblk = pair_blocks(qp, qo, nkb);
        const int nc = (nblk + chunk - 1) / chunk;
        for (int c = 0; c < nc; ++c) {
            const int len = std::min((c + 1) * chunk, nblk) - c * chunk;
            it.push_back({len + 1.0f + (nc > 1 ? 3.0f : 0.f), (static_cast<uint32_t>(qp) << 16) | c});
        }
    }
    std::stable_sort(it.begin(), it.end(), [](const auto& a, const auto& b) {
        return a.first > b.first || (a.first == b.first && a.second > b.second);
    });
    std::priority_queue<double, std::vector<double>, std::greater<double>> load;
    for (int i = 0; i < sms; ++i) load.push(0.0);
    double span = 0.0;
    for (const auto& e : it)
        for (int hh = 0; hh < nq; ++hh) {
            const double t = load.top() + e.first;
            load.pop();
            load.push(t);
            span = std::max(span, t);
        }
    if (out) *out = std::move(it);
    return span;
}

// T: query rows, T_kv: key rows, qo: query offset in 128-blocks
const FwdSplit& fwd_split_plan(int T, int nq, int T_kv, int qo) {
    static std::map<std::tuple<int, int, int, int>, FwdSplit> cache;  // nodes are stable: references stay valid
    static std::mutex mu;  // loopback groups launch from several host threads
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_tuple(T, nq, T_kv, qo);
    auto f = cache.find(key);
    if (f != cache.end()) return f->second;
    FwdSplit sp;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int nkb = (T_kv + BKV - 1) / BKV;
    const int npairs = ((T + BQ - 1) / BQ + 1) / 2;
    // many heads x pairs per SM already balance; only small grids are split
    // (measured on B200: 16 heads x 16 pairs, 1.7 items per SM, run faster unsplit)
    if (2LL * nq * npairs > 3LL * sms) return cache.emplace(key, sp).first->second;
    const int full = pair_blocks(npairs - 1, qo, nkb);  // the longest row
    double best = fwd_makespan(nq, npairs, qo, nkb, full, sms, nullptr);
    // DH_ATTN_FWD_CHUNK=<even KV blocks> forces a chunk size (tuning runs)
    const char* force = std::getenv("DH_ATTN_FWD_CHUNK");
    const int forced = force ? std::atoi(force) : 0;
    for (int div : {2, 3, 4, 6, 8}) {
        const int c = forced ? forced : std::max(2, 2 * ((full + 2 * div - 1) / (2 * div)));
        if (c >= full || (full + c - 1) / c > 16 || c % 2) continue;
        std::vector<std::pair<float, uint32_t>> it;
        const double ms = fwd_makespan(nq, npairs, qo, nkb, c, sms, &it);
        if ((forced || ms < 0.85 * best) && static_cast<int>(it.size()) <= kMaxItems) {
            best = ms;
            sp.chunk = c;
            sp.maxc = (full + c - 1) / c;
            sp.items = static_cast<int>(it.size());
            for (size_t i = 0; i < it.size(); ++i) sp.sched.item[i] = it[i].second;
        }
    }
    return cache.emplace(key, sp).first->second;
}

}  // namespace

long long attn_fwd_tc_scratch_floats(int T, int nq, int D, int T_kv, int q_offset) {
    const FwdSplit& sp = fwd_split_plan(T, nq, T_kv, q_offset / BQ);
    if (!sp.chunk) return 0;
    const long long nqb2 = 2LL * (((T + BQ - 1) / BQ + 1) / 2);
    return static_cast<long long>(nq) * nqb2 * sp.maxc * (BQ * D + 2 * BQ);
}

namespace {

template <int D>
int attn_fwd_tc_d(const void* q, const void* k, const void* v, long long ldq, long long ldkv, void* o,
                  long long ldo, float* lse, int T, int nq, int nkv, float scale, float* scratch,
                  long long scratch_floats, int T_kv, int q_offset, cudaStream_t s) {
    CUtensorMap mq, mk, mv;
    int rc = make_tma_2d(&mq, q, static_cast<long long>(nq) * D, T, ldq, 64, BQ);
    if (rc) return rc;
    rc = make_tma_2d(&mk, k, static_cast<long long>(nkv) * D, T_kv, ldkv, 64, BKV);
    if (rc) return rc;
    rc = make_tma_2d(&mv, v, static_cast<long long>(nkv) * D, T_kv, ldkv, 64, BKV);
    if (rc) return rc;
    static bool cfg = false;
    if (!cfg) {
        DH_CUDA_CHECK(cudaFuncSetAttribute(attn_fwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           FwdSmem<D>::total));
        cfg = true;
    }
    const int nkb = (T_kv + BKV - 1) / BKV;
    const int npairs = ((T + BQ - 1) / BQ + 1) / 2;
    const int qo = q_offset / BQ;
    FwdParams prm{lse, static_cast<__nv_bfloat16*>(o), ldo, T, nq / nkv, scale * kLog2e, nq, nkb, npairs, 0, 1,
                  scratch, T_kv, qo};
    const FwdSplit& sp = fwd_split_plan(T, nq, T_kv, qo);
    const bool split =
        sp.chunk && scratch && scratch_floats >= attn_fwd_tc_scratch_floats(T, nq, D, T_kv, q_offset);
    if (split) {
        prm.chunk = sp.chunk;
        prm.maxc = sp.maxc;
    }
    const int grid = (split ? sp.items : npairs) * nq;
    attn_fwd_tc_kernel<D><<<grid, kThreads, FwdSmem<D>::total, s>>>(mq, mk, mv, prm, sp.sched);
    DH_CUDA_CHECK(cudaGetLastError());
    if (split) {
        const dim3 cg(2 * npairs, nq, combine_slices<D>());
        if (sp.maxc <= 2) attn_fwd_combine_kernel<2, D><<<cg, 256, 0, s>>>(prm);
        else if (sp.maxc <= 4) attn_fwd_combine_kernel<4, D><<<cg, 256, 0, s>>>(prm);
        else if (sp.maxc <= 8) attn_fwd_combine_kernel<8, D><<<cg, 256, 0, s>>>(prm);
        else attn_fwd_combine_kernel<16, D><<<cg, 256, 0, s>>>(prm);
        DH_CUDA_CHECK(cudaGetLastError());
    }
    return DH_OK;
}

}  // namespace

// Host launcher (dh_attn_fwd dispatches here for head_dim 64 and 128). T
// query rows at global positions [q_offset, q_offset + T) attend causally to
// T_kv key rows (context parallelism: q_offset = rank * T, keys gathered).
int attn_fwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv, void* o,
                long long ldo, float* lse, int T, int nq, int nkv, int D, float scale, float* scratch,
                long long scratch_floats, int T_kv, int q_offset, cudaStream_t s) {
    if (q_offset % (2 * BQ) || q_offset + T > T_kv)
        return set_error(DH_ERR_INVALID, "attn: q_offset must be a multiple of 256 and q_offset + T <= T_kv");
    if (D == 128)
        return attn_fwd_tc_d<128>(q, k, v, ldq, ldkv, o, ldo, lse, T, nq, nkv, scale, scratch, scratch_floats, T_kv,
                                  q_offset, s);
    if (D == 64)
        return attn_fwd_tc_d<64>(q, k, v, ldq, ldkv, o, ldo, lse, T, nq, nkv, scale, scratch, scratch_floats, T_kv,
                                 q_offset, s);
    return set_error(DH_ERR_INVALID, "attn: head_dim must be 64 or 128");
}

}  // namespace dh

// ===========================================================================
// Backward (attn_bwd node): one launch, two deterministic tcgen05 work kinds.
// Every MMA has N >= 128: at M = 128 a tcgen05.mma with N = 64 takes ~51
// cycles per K = 16 step against 64 at N = 128 (tools/micro/mma_rate.cu on
// B200: N = 32 / 64 reach 0.31 / 0.62 of the dense rate, N >= 128 1.00), so
// both kinds use 128-row tiles and single-buffered S / dP in TMEM, with the
// MMA issue order arranged so the tensor pipe never waits on the elementwise
// warps in steady state (see each body).
//
// dK/dV item — one CTA per (128-key block, q head); inner q tiles of 128:
//   S^T  = K Q^T        M128 N128 K=D   A=K (smem)      B=Q (smem, K-major)
//   dP^T = V dO^T       M128 N128 K=D   A=V (smem)      B=dO (smem, K-major)
//   P^T = exp(scale S^T - lse_q), dS^T = P^T (dP^T - D_q)      (thread = key row)
//   dV  += P^T dO       M128 N=D K128   A=P^T (TMEM)    B=dO (smem, MN-major)
//   dK  += dS^T Q       M128 N=D K128   A=dS^T (TMEM)   B=Q  (smem, MN-major)
//   TMEM: S^T (128) | dP^T (128) | dV (D) | dK (D); P^T / dS^T (bf16 pairs)
//   overwrite the first kEwCols / 2 columns of each kEwCols-column part of
//   S^T / dP^T that the same threads read (no cross-thread hazard).
//   Issue order: S(0) dP(0) | dV(i) S(i+1) dK(i) dP(i+1) | ... — the softmax
//   exponentials of tile i+1 run under dK(i) and dP(i+1), dS(i) under dV(i)
//   and S(i+1).
// dQ item — one CTA per (128-query block, q head); inner key tiles of 128:
//   S = Q K^T, dP = dO V^T (M128 N128 K=D, A = Q / dO resident in TMEM),
//   dS = P (dP - D)    (thread = query row)
//   dQ += dS K          M128 N=D K128   A=dS (TMEM)     B=K (smem, MN-major)
//   TMEM: S (128) | dP (128) | dQ (D) | Q (D/2) | dO (D/2).
//   Issue order: S(0) dP(0) | S(i+1) dQ(i) dP(i+1) | ... — S(i+1) is issued as
//   soon as the elementwise warps have read S(i) into registers.
// Work items come from a host plan (bwd_plan): with few heads per GPU (high
// TP) the longest causal items would be the critical path, so items costlier
// than the per-SM average are split into chunks of their inner loop (q tiles
// of a dK/dV item, key tiles of a dQ item), dispatched heaviest first. No
// atomics: an item writes bf16 directly when it alone owns its output rows;
// otherwise (GQA group > 1, or split) it writes an fp32 partial slot and
// attn_bwd_reduce sums the slots in a fixed (head, chunk) order.
// ===========================================================================

namespace dh {
namespace {

// The Q ring is one stage deeper than the dO ring: a Q slot is refilled after
// dK(i) and read again by S^T(i + kQS), so at D = 128 (three Q stages, two dO
// stages, 227 KB exactly) every refill has five to six MMAs (> 2.5k cycles) to
// land. Small vectors and barriers come first, the 1024-aligned tiles after
// them: this layout needs a 1024-aligned dynamic shared memory base (checked).
template <int D>
struct KvSmem {
    static constexpr int kTile = tile_bytes<D>();         // 128-row tile
    static constexpr int kQS = D == 128 ? 3 : 4;          // Q ring stages (+ lse rows)
    static constexpr int kOS = D == 128 ? 2 : 4;          // dO ring stages (+ D rows)
    static constexpr int lse = 0;                         // [kQS][128] fp32 (raw lse)
    static constexpr int dvec = lse + kQS * 512;          // [kOS][128] fp32
    static constexpr int bars = dvec + kOS * 512;
    static constexpr int k = (bars + 256 + 1023) / 1024 * 1024;
    static constexpr int v = k + kTile;
    static constexpr int q = v + kTile;                   // kQS tiles
    static constexpr int dout = q + kQS * kTile;          // kOS tiles
    static constexpr int total = dout + kOS * kTile;
};

template <int D>
struct DqSmem {
    static constexpr int kTile = tile_bytes<D>();
    static constexpr int kSt = D == 128 ? 3 : 6;          // K/V ring stages (Q and dO live in TMEM)
    static constexpr int k = 0;                           // kSt tiles
    static constexpr int v = k + kSt * kTile;             // kSt tiles
    static constexpr int bars = v + kSt * kTile;
    static constexpr int total = bars + 256 + 1024;
};
static_assert(KvSmem<128>::total <= 232448 && DqSmem<128>::total <= 232448, "backward smem exceeds the sm_100 limit");
static_assert(KvSmem<64>::total <= 232448 && DqSmem<64>::total <= 232448, "backward smem exceeds the sm_100 limit");

struct BwdParams {
    const __nv_bfloat16* q;     // raw rows for the TMEM-resident Q / dO of the dQ items
    const __nv_bfloat16* dout;
    long long ldq, ldo;
    const float* lse;
    const float* dvec;
    float* dk_part;             // [slot][128 keys][D] fp32 (scaled)
    float* dv_part;
    float* dq_part;             // [slot][128 queries][D] fp32 (scaled)
    __nv_bfloat16* dk;
    __nv_bfloat16* dv;
    __nv_bfloat16* dq;
    long long lddkv, lddq;
    int T, group;   // T: query rows (this rank's)
    int hpi;        // q heads per dK/dV item: 1, or the GQA group (its heads accumulate into
                    // one dK / dV in TMEM, no partial slots; TP = 1 shapes, see bwd_plan)
    float scale, scale_log2;
    int T_kv;       // key rows
    int qo;         // query offset in 128-blocks (context parallelism), even
};

// Elementwise warps of the backward kernel: kEwWarps / 4 per TMEM lane
// quadrant, each owning kEwCols of the 128 tile columns. 16 (4 per quadrant,
// 32 columns each) halves the per-thread latency of the exp / dS phases that
// sit between the MMA groups (8 warps: 64 columns each); the per-SM MUFU and
// FMA work is the same.
#ifndef DH_ATTN_BWD_EW
#define DH_ATTN_BWD_EW 8
#endif
constexpr int kEwWarps = DH_ATTN_BWD_EW;
static_assert(kEwWarps == 8 || kEwWarps == 16, "elementwise warps: 2 or 4 per TMEM quadrant");
constexpr int kEwParts = kEwWarps / 4;          // column parts per lane quadrant
constexpr int kEwCols = 128 / kEwParts;         // tile columns per elementwise thread
constexpr int kEwThreads = 32 * kEwWarps;
constexpr int kEw0 = 2;                              // first elementwise warp
constexpr int kThreadsBwd = 32 * kEw0 + kEwThreads;  // producer, MMA issuer, elementwise warps
constexpr uint32_t kDirect = 0xFFFFFFFFu;  // item owns its output rows: bf16 store, no slot

// Explicit schedule (kernel parameter): item.x = kind << 31 (1 = dQ) | head << 24
// | block << 16 | c0 << 8 | c1, item.y = partial slot or kDirect; heaviest first.
constexpr int kMaxBwdItems = 2900;
struct BwdSched {
    int n;  // 0: implicit rank order, no splits (see attn_bwd_tc_kernel)
    uint2 item[kMaxBwdItems];
};
// Partial-slot tables of the reduction: slot of (head h, block b, chunk c) =
// base[b] + h * nck[b] + c, so a GQA group's heads and a block's chunks are
// contiguous and summed in that order.
constexpr int kMaxBwdBlocks = 256;
struct BwdSlots {
    uint32_t kv_base[kMaxBwdBlocks], q_base[kMaxBwdBlocks];  // kDirect: no partials for the block
    uint8_t kv_nck[kMaxBwdBlocks], q_nck[kMaxBwdBlocks];
};

// A operand from TMEM (bf16 pairs) for k-step kk (16 rows of the 128-wide
// tile): each kEwCols-column part of the fp32 tile holds its values packed
// into its first kEwCols / 2 columns (by the thread that read them).
__device__ __forceinline__ uint32_t packed_col(int kk) {
    constexpr int kps = kEwCols / 16;  // k-steps per part
    return (kk / kps) * kEwCols + (kk % kps) * 8;
}

// N consecutive fp32 columns of this warp's TMEM lane quadrant (waited).
template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, uint32_t (&r)[N]) {
    static_assert(N % 16 == 0, "16-column granules");
    if constexpr (N % 32 == 0) {
#pragma unroll
        for (int c = 0; c < N / 32; ++c) tmem_ld32(taddr + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]));
    } else {
#pragma unroll
        for (int c = 0; c < N / 16; ++c) tmem_ld16(taddr + 16 * c, *reinterpret_cast<uint32_t(*)[16]>(&r[16 * c]));
    }
    tmem_ld_wait();
}
template <int N>
__device__ __forceinline__ void tmem_stn(uint32_t taddr, const uint32_t (&r)[N]) {
    static_assert(N % 16 == 0, "16-column granules");
    if constexpr (N % 32 == 0) {
#pragma unroll
        for (int c = 0; c < N / 32; ++c)
            tmem_st32(taddr + 32 * c, *reinterpret_cast<const uint32_t(*)[32]>(&r[32 * c]));
    } else {
#pragma unroll
        for (int c = 0; c < N / 16; ++c)
            tmem_st16(taddr + 16 * c, *reinterpret_cast<const uint32_t(*)[16]>(&r[16 * c]));
    }
}

// p = 2^(s * scale_log2 + bias), bias per column (-log2e lse_j, PER_COL) or
// per row; DH_ATTN_BWD_POLY_Q quarters of the pairs on the FMA pipe. The
// split barely matters (attention bench, TP=1 bwd: 0.401 ms for a quarter,
// 0.405 for a half or none, 0.419 for three quarters): the exp phase is not
// MUFU-bound (profiles/r02_attn_bwd_investigation.txt).
template <bool PER_COL, int N>
__device__ __forceinline__ void bwd_exp(uint32_t (&s)[N], const float* bias, float bias_row, float scale_log2) {
    const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
#pragma unroll
    for (int u = 0; u < N / 2; ++u) {
        uint64_t b2;
        if constexpr (PER_COL) {  // bias = raw lse of the columns (smem): -log2e * lse
            const float2 l2 = reinterpret_cast<const float2*>(bias)[u];
            b2 = ffma2(f2_pack(l2.x, l2.y), f2_pack(-kLog2e, -kLog2e), 0ull);
        } else {
            b2 = f2_pack(bias_row, bias_row);
        }
        const uint64_t x = ffma2(f2_pack(__uint_as_float(s[2 * u]), __uint_as_float(s[2 * u + 1])), sc2, b2);
        float x0, x1;
        f2_unpack(x, x0, x1);
        float e0, e1;
        if (DH_ATTN_POLY && (u & 3) >= 4 - DH_ATTN_BWD_POLY_Q) {
            f2_unpack(exp2_fma2(x0, x1), e0, e1);
        } else {
            e0 = fast_exp2(x0);
            e1 = fast_exp2(x1);
        }
        s[2 * u] = __float_as_uint(e0);
        s[2 * u + 1] = __float_as_uint(e1);
    }
}

// dS = P (dP - D), packed to bf16 pairs over the first N / 2 columns read.
template <bool PER_COL, int N>
__device__ __forceinline__ void bwd_ds_store(uint32_t taddr, const uint32_t (&pv)[N], const float* dcol, uint64_t nd_row) {
    uint32_t b[N];
    tmem_ldn<N>(taddr, b);
    uint32_t pd[N / 2];
#pragma unroll
    for (int u = 0; u < N / 2; ++u) {
        uint64_t nd = nd_row;
        if constexpr (PER_COL) {
            const float2 dd = reinterpret_cast<const float2*>(dcol)[u];
            nd = f2_pack(-dd.x, -dd.y);
        }
        const uint64_t ds = ffma2(f2_pack(__uint_as_float(pv[2 * u]), __uint_as_float(pv[2 * u + 1])),
                                  fadd2(f2_pack(__uint_as_float(b[2 * u]), __uint_as_float(b[2 * u + 1])), nd), 0ull);
        float s0, s1;
        f2_unpack(ds, s0, s1);
        pd[u] = pack2(s0, s1);
    }
    tmem_stn<N / 2>(taddr, pd);
}

// ptxas spills two scalars of this body (the item's slot and kv head, 12 bytes,
// read once in the epilogue); re-reading them from shared memory instead
// removes the spill but measured 1-2% slower (register allocation of the loop).
template <int D>
__device__ __forceinline__ void attn_bwd_dkdv_body(const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                                                   const CUtensorMap& tm_q, const CUtensorMap& tm_do,
                                                   const BwdParams& p, const int kb, const int h, const int c0,
                                                   const int c1, const uint32_t slot) {
    using Smem = dh::KvSmem<D>;
    constexpr int kTile = Smem::kTile, kQS = Smem::kQS, kOS = Smem::kOS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw;  // 1024-aligned (see KvSmem)
    if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u)) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Smem::bars);
    uint64_t* kv_full = bars + 0;
    uint64_t* q_full = bars + 1;                // [kQS] Q ring (+ lse)
    uint64_t* q_empty = q_full + kQS;           // [kQS]
    uint64_t* o_full = q_empty + kQS;           // [kOS] dO ring (+ D)
    uint64_t* o_empty = o_full + kOS;           // [kOS]
    uint64_t* s_full = o_empty + kOS;           // S^T in TMEM
    uint64_t* dp_full = s_full + 1;             // dP^T in TMEM
    uint64_t* p_full = dp_full + 1;             // P^T (bf16) in TMEM
    uint64_t* ds_full = p_full + 1;             // dS^T (bf16) in TMEM
    uint64_t* acc_done = ds_full + 1;           // dK/dV complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);
    float* lse_s = reinterpret_cast<float*>(sm + Smem::lse);    // [kQS][128]
    float* dvec_s = reinterpret_cast<float*>(sm + Smem::dvec);  // [kOS][128]

    const int kvh = h / p.group;
    // q tiles [c0, c1) of the tiles from the first one with a query at or after
    // the block's first key (c1 < 0: all of them), for p.hpi consecutive q heads
    // from h (iteration it: head h + it / n_head, tile i0 + it % n_head)
    const int nq128 = (p.T + BQ - 1) / BQ;
    const int i0 = max(0, kb - p.qo) + c0;
    const int n_head = c1 < 0 ? max(0, nq128 - i0) : c1 - c0;
    const int n_it = n_head * p.hpi;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        mbar_init(kv_full, 1);
        for (int i = 0; i < kQS; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < kOS; ++i) {
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(dp_full, 1);
        mbar_init(p_full, kEwThreads);
        mbar_init(ds_full, kEwThreads);
        mbar_init(acc_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t t_s = tmem, t_dp = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 256 + D;
    const bool bulk_vec = (p.T % BQ) == 0;  // lse / D rows fetched by bulk copy

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(kv_full, 2 * kTile);
#pragma unroll
            for (int hh = 0; hh < D / 64; ++hh) {
                tma_load_2d(sm + Smem::k + hh * kHalf, &tm_k, kv_full, kvh * D + 64 * hh, kb * BKV);
                tma_load_2d(sm + Smem::v + hh * kHalf, &tm_v, kv_full, kvh * D + 64 * hh, kb * BKV);
            }
            for (int it = 0; it < n_it; ++it) {
                const int qs = it % kQS, os = it % kOS, qi = i0 + it % n_head, hq = h + it / n_head;
                const long long off = static_cast<long long>(hq) * p.T + qi * BQ;
                // Q(it), dO(it) and their vectors all complete on q_full[qs]: the
                // MMA thread waits once per iteration for its TMA operands (each
                // wait between MMA groups costs the tensor pipe ~150 cycles on
                // B200, tools/micro/mma_rate.cu); the two rings keep separate
                // empty barriers (different depths)
                mbar_wait(&q_empty[qs], ((it / kQS) & 1) ^ 1);
                mbar_expect_tx(&q_full[qs], 2 * kTile + (bulk_vec ? 1024 : 0));
                if (bulk_vec) bulk_load_1d(lse_s + qs * 128, p.lse + off, 512, &q_full[qs]);
#pragma unroll
                for (int hh = 0; hh < D / 64; ++hh)
                    tma_load_2d(sm + Smem::q + qs * kTile + hh * kHalf, &tm_q, &q_full[qs], hq * D + 64 * hh, qi * BQ);
                mbar_wait(&o_empty[os], ((it / kOS) & 1) ^ 1);
                if (bulk_vec) bulk_load_1d(dvec_s + os * 128, p.dvec + off, 512, &q_full[qs]);
#pragma unroll
                for (int hh = 0; hh < D / 64; ++hh)
                    tma_load_2d(sm + Smem::dout + os * kTile + hh * kHalf, &tm_do, &q_full[qs], hq * D + 64 * hh,
                                qi * BQ);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_s = umma_idesc_bf16(128, 128, false, false);
        constexpr uint32_t id_g = umma_idesc_bf16(128, D, false, true);
        const uint32_t k_addr = smem_u32(sm + Smem::k), v_addr = smem_u32(sm + Smem::v);
        auto q_addr = [&](int it) { return smem_u32(sm + Smem::q + (it % kQS) * kTile); };
        auto o_addr = [&](int it) { return smem_u32(sm + Smem::dout + (it % kOS) * kTile); };
        auto issue_s = [&](int it) {  // S^T(it) = K Q(it)^T; Q(it) and dO(it) landed
            mbar_wait(&q_full[it % kQS], (it / kQS) & 1);
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    tc_mma_bf16(t_s, desc_kmajor(k_addr, kk), desc_kmajor(q_addr(it), kk), id_s, kk > 0);
                tc_commit(s_full);
            }
            __syncwarp();
        };
        auto issue_dp = [&](int it) {  // dP^T(it) = V dO(it)^T (dO(it) waited with Q(it) in issue_s)
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    tc_mma_bf16(t_dp, desc_kmajor(v_addr, kk), desc_kmajor(o_addr(it), kk), id_s, kk > 0);
                tc_commit(dp_full);
            }
            __syncwarp();
        };
        mbar_wait(kv_full, 0);
        if (n_it > 0) {
            issue_s(0);
            issue_dp(0);
        }
        for (int it = 0; it < n_it; ++it) {
            // dV += P^T(it) dO(it)
            if (lane == 0) ATR(it * 8 + 0);
            mbar_wait(p_full, it & 1);
            if (lane == 0) ATR(it * 8 + 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < BQ / 16; ++kk)
                    tc_mma_bf16_ts(t_dv, t_s + packed_col(kk), desc_mnmajor(o_addr(it), kk), id_g, (it | kk) != 0);
            }
            __syncwarp();
            // S^T(it+1) overwrites P^T(it): the dV MMAs above were issued first
            if (it + 1 < n_it) issue_s(it + 1);
            // dK += dS^T(it) Q(it)
            mbar_wait(ds_full, it & 1);
            if (lane == 0) ATR(it * 8 + 2);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < BQ / 16; ++kk)
                    tc_mma_bf16_ts(t_dk, t_dp + packed_col(kk), desc_mnmajor(q_addr(it), kk), id_g, (it | kk) != 0);
                // dK(it) is the last reader of Q(it) and of the lse / D rows the
                // elementwise warps used (they arrived on ds_full first)
                tc_commit(&q_empty[it % kQS]);
                tc_commit(&o_empty[it % kOS]);
                if (it + 1 == n_it) tc_commit(acc_done);
            }
            __syncwarp();
            // dP^T(it+1) overwrites dS^T(it): the dK MMAs above were issued first
            if (it + 1 < n_it) issue_dp(it + 1);
        }
    } else {
        // quadrant (TMEM lanes) = warp & 3, column part = (warp - kEw0) >> 2
        const int quad = warp & 3;
        const int part = (warp - kEw0) >> 2;
        const int r = quad * 32 + lane;  // key row within the block
        const int key = kb * BKV + r;
        const int t_sm = threadIdx.x - 32 * kEw0;  // among the elementwise warps
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t col = lane_off + part * kEwCols;
        const int key_hi = kb * BKV + BKV - 1;
        for (int it = 0; it < n_it; ++it) {
            const int qi = i0 + it % n_head, hq = h + it / n_head;
            float* sl = lse_s + (it % kQS) * 128;
            float* sd = dvec_s + (it % kOS) * 128;
            if (!bulk_vec) {
                // ragged T: stage the vectors with plain loads
                named_barrier(1, kEwThreads);  // previous readers of these slots are done
                if (t_sm < BQ) {
                    const int q = qi * BQ + t_sm;
                    sl[t_sm] = q < p.T ? p.lse[static_cast<long long>(hq) * p.T + q] : 0.f;
                    sd[t_sm] = q < p.T ? p.dvec[static_cast<long long>(hq) * p.T + q] : 0.f;
                }
                named_barrier(1, kEwThreads);
            }
            // whole tile causal-visible and in range: no per-element masking
            const int qg0 = (p.qo + qi) * BQ;  // global position of the tile's first query
            const bool full_tile = qg0 >= key_hi && qi * BQ + BQ <= p.T && key_hi < p.T_kv;
            // ---- P^T = exp2(scale_log2 S^T - log2e lse_q)
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 7);
            mbar_wait(s_full, it & 1);
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 3);
            tc_fence_after();
            uint32_t pv[kEwCols];
            tmem_ldn<kEwCols>(t_s + col, pv);
            bwd_exp<true>(pv, sl + part * kEwCols, 0.f, p.scale_log2);
            if (!full_tile) {
#pragma unroll
                for (int j = 0; j < kEwCols; ++j) {
                    const int q = qi * BQ + part * kEwCols + j;  // local row; global position q + qo * BQ
                    if (q + p.qo * BQ < key || q >= p.T || key >= p.T_kv) pv[j] = 0u;
                }
            }
            {
                uint32_t pp[kEwCols / 2];
#pragma unroll
                for (int u = 0; u < kEwCols / 2; ++u)
                    pp[u] = pack2(__uint_as_float(pv[2 * u]), __uint_as_float(pv[2 * u + 1]));
                tmem_stn<kEwCols / 2>(t_s + col, pp);
            }
            tmem_st_wait();
            tc_fence_before();
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 4);
            mbar_arrive(p_full);
            // ---- dS^T = P^T (dP^T - D_q)
            mbar_wait(dp_full, it & 1);
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 5);
            tc_fence_after();
            bwd_ds_store<true>(t_dp + col, pv, sd + part * kEwCols, 0ull);
            tmem_st_wait();
            tc_fence_before();
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 6);
            mbar_arrive(ds_full);
        }
        if (n_it > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        const bool ok = key < p.T_kv;
        constexpr int kPc = D / kEwParts;          // dK / dV columns per part
        constexpr int kW = kPc < 32 ? kPc : 32;    // per TMEM load
#pragma unroll 1
        for (int c = part * kPc; c < (part + 1) * kPc; c += kW) {
            uint32_t ka[kW], va[kW];
            tmem_ldn<kW>(t_dk + lane_off + c, ka);
            tmem_ldn<kW>(t_dv + lane_off + c, va);
            if (!ok) continue;
            if (slot == kDirect) {
                __nv_bfloat16* kr = p.dk + static_cast<long long>(key) * p.lddkv + kvh * D + c;
                __nv_bfloat16* vr = p.dv + static_cast<long long>(key) * p.lddkv + kvh * D + c;
#pragma unroll
                for (int t = 0; t < kW; t += 8) {
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
                float* kr = p.dk_part + (static_cast<long long>(slot) * BKV + r) * D + c;
                float* vr = p.dv_part + (static_cast<long long>(slot) * BKV + r) * D + c;
                // keys after every query of this rank (context parallelism) get no
                // gradient; TMEM was never written for them (select, not multiply)
                const bool any = n_it > 0;
#pragma unroll
                for (int t = 0; t < kW; t += 4) {
                    float k4[4], v4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        k4[u] = any ? __uint_as_float(ka[t + u]) * p.scale : 0.f;
                        v4[u] = any ? __uint_as_float(va[t + u]) : 0.f;
                    }
                    *reinterpret_cast<float4*>(kr + t) = make_float4(k4[0], k4[1], k4[2], k4[3]);
                    *reinterpret_cast<float4*>(vr + t) = make_float4(v4[0], v4[1], v4[2], v4[3]);
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

template <int D>
__device__ __forceinline__ void attn_bwd_dq_body(const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                                                 const BwdParams& p, const int qb, const int h, const int c0,
                                                 const int c1, const uint32_t slot) {
    using Smem = dh::DqSmem<D>;
    constexpr int kTile = Smem::kTile, kSt = Smem::kSt;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Smem::bars);
    uint64_t* q_full = bars + 0;           // Q / dO rows stored into TMEM
    uint64_t* kv_full = bars + 1;          // [kSt] K/V ring
    uint64_t* kv_empty = kv_full + kSt;    // [kSt]
    uint64_t* s_full = kv_empty + kSt;
    uint64_t* dp_full = s_full + 1;
    uint64_t* s_free = dp_full + 1;        // S read into registers
    uint64_t* ds_full = s_free + 1;        // dS (bf16) in TMEM
    uint64_t* acc_done = ds_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

    const int kvh = h / p.group;
    // key tiles [c0, c1) of those covering the block's last query (global
    // position); c1 < 0: all of them. `it` below counts from c0.
    const int n_it = (c1 < 0 ? min(p.qo + qb + 1, (p.T_kv + BKV - 1) / BKV) : c1) - c0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        mbar_init(q_full, kEwThreads);
        for (int i = 0; i < kSt; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(dp_full, 1);
        mbar_init(s_free, kEwThreads);
        mbar_init(ds_full, kEwThreads);
        mbar_init(acc_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // S | dP | dQ | Q (bf16 pairs) | dO (bf16 pairs): Q and dO are the A
    // operands of every S / dP MMA, so they are read from TMEM, not shared memory
    const uint32_t t_s = tmem, t_dp = tmem + 128, t_dq = tmem + 256, t_qa = tmem + 384,
                   t_doa = tmem + 384 + D / 2;

    if (warp == 0) {
        if (lane == 0) {
            for (int it = 0; it < n_it; ++it) {
                const int st = it % kSt;
                mbar_wait(&kv_empty[st], ((it / kSt) & 1) ^ 1);
                mbar_expect_tx(&kv_full[st], 2 * kTile);
                uint8_t* kd = sm + Smem::k + st * kTile;
                uint8_t* vd = sm + Smem::v + st * kTile;
#pragma unroll
                for (int hh = 0; hh < D / 64; ++hh) {
                    tma_load_2d(kd + hh * kHalf, &tm_k, &kv_full[st], kvh * D + 64 * hh, (c0 + it) * BKV);
                    tma_load_2d(vd + hh * kHalf, &tm_v, &kv_full[st], kvh * D + 64 * hh, (c0 + it) * BKV);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_s = umma_idesc_bf16(128, 128, false, false);
        constexpr uint32_t id_g = umma_idesc_bf16(128, D, false, true);
        auto k_addr = [&](int it) { return smem_u32(sm + Smem::k + (it % kSt) * kTile); };
        auto v_addr = [&](int it) { return smem_u32(sm + Smem::v + (it % kSt) * kTile); };
        auto issue_s = [&](int it) {  // S(it) = Q K(it)^T (TMA operands: no tcgen05 fence, as CUTLASS)
            mbar_wait(&kv_full[it % kSt], (it / kSt) & 1);
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    tc_mma_bf16_ts(t_s, t_qa + kk * 8, desc_kmajor(k_addr(it), kk), id_s, kk > 0);
                tc_commit(s_full);
            }
            __syncwarp();
        };
        auto issue_dp = [&](int it) {  // dP(it) = dO V(it)^T (stage already waited)
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    tc_mma_bf16_ts(t_dp, t_doa + kk * 8, desc_kmajor(v_addr(it), kk), id_s, kk > 0);
                tc_commit(dp_full);
            }
            __syncwarp();
        };
        mbar_wait(q_full, 0);
        tc_fence_after();
        issue_s(0);
        issue_dp(0);
        for (int it = 0; it < n_it; ++it) {
            if (lane == 0) ATR(it * 8 + 0);
            if (it + 1 < n_it) {
                mbar_wait(s_free, it & 1);  // S(it) is in registers
                if (lane == 0) ATR(it * 8 + 1);
                issue_s(it + 1);
            }
            mbar_wait(ds_full, it & 1);
            if (lane == 0) ATR(it * 8 + 2);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk)
                    tc_mma_bf16_ts(t_dq, t_dp + packed_col(kk), desc_mnmajor(k_addr(it), kk), id_g, (it | kk) != 0);
                tc_commit(&kv_empty[it % kSt]);
                if (it + 1 == n_it) tc_commit(acc_done);
            }
            __syncwarp();
            // dP(it+1) overwrites dS(it): the dQ MMAs above were issued first
            if (it + 1 < n_it) issue_dp(it + 1);
        }
    } else {
        const int quad = warp & 3;
        const int part = (warp - kEw0) >> 2;
        const int r = quad * 32 + lane;
        const int qrow = qb * BQ + r;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t col = lane_off + part * kEwCols;
        const int qc = min(qrow, p.T - 1);
        const float nlse2 = -p.lse[static_cast<long long>(h) * p.T + qc] * kLog2e;
        const float dd = p.dvec[static_cast<long long>(h) * p.T + qc];
        const uint64_t nd2 = f2_pack(-dd, -dd);
        {
            // this thread's query row of Q (first half of the parts) or dO (second
            // half) into its TMEM lane: row-major bf16 pairs are exactly the packed
            // A-operand columns; each part stages D / kEwParts pair columns
            constexpr int kSub = kEwParts / 2;            // parts per operand
            constexpr int kPw = D / 2 / kSub;             // pair columns per part
            constexpr int kW = kPw < 32 ? kPw : 32;       // per TMEM store
            const bool is_do = part >= kSub;
            const int sub = part % kSub;
            const __nv_bfloat16* src = is_do ? p.dout + static_cast<long long>(qc) * p.ldo + h * D
                                             : p.q + static_cast<long long>(qc) * p.ldq + h * D;
            const bool in = qrow < p.T;
#pragma unroll
            for (int c = sub * kPw; c < (sub + 1) * kPw; c += kW) {
                uint32_t w[kW];
#pragma unroll
                for (int u = 0; u < kW / 4; ++u) {
                    const uint4 x = in ? *reinterpret_cast<const uint4*>(src + 2 * c + u * 8) : make_uint4(0, 0, 0, 0);
                    w[4 * u] = x.x;
                    w[4 * u + 1] = x.y;
                    w[4 * u + 2] = x.z;
                    w[4 * u + 3] = x.w;
                }
                tmem_stn<kW>((is_do ? t_doa : t_qa) + lane_off + c, w);
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(q_full);
        }
        const int qpos = (p.qo + qb) * BQ + r;  // this row's global query position
        for (int it = 0; it < n_it; ++it) {
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 7);
            mbar_wait(s_full, it & 1);
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 3);
            tc_fence_after();
            uint32_t pv[kEwCols];
            tmem_ldn<kEwCols>(t_s + col, pv);
            tc_fence_before();
            mbar_arrive(s_free);
            const int qg0 = (p.qo + qb) * BQ;  // global position of the block's first query
            const int kt = c0 + it;  // absolute key tile
            const bool full_tile = kt * BKV + BKV - 1 <= qg0 && kt * BKV + BKV <= p.T_kv && qb * BQ + BQ <= p.T;
            bwd_exp<false>(pv, nullptr, nlse2, p.scale_log2);
            if (!full_tile) {
#pragma unroll
                for (int j = 0; j < kEwCols; ++j) {
                    const int key = kt * BKV + part * kEwCols + j;
                    if (key > qpos || key >= p.T_kv) pv[j] = 0u;
                }
            }
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 4);
            mbar_wait(dp_full, it & 1);
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 5);
            tc_fence_after();
            bwd_ds_store<false>(t_dp + col, pv, nullptr, nd2);
            tmem_st_wait();
            tc_fence_before();
            if (threadIdx.x == 32 * kEw0) ATR(it * 8 + 6);
            mbar_arrive(ds_full);
        }
        mbar_wait(acc_done, 0);
        tc_fence_after();
        const bool ok = qrow < p.T;
        __nv_bfloat16* row = p.dq + static_cast<long long>(qrow) * p.lddq + h * D;
        float* prow = p.dq_part + (static_cast<long long>(slot) * BQ + r) * D;
        constexpr int kPc = D / kEwParts;          // dQ columns per part
        constexpr int kW = kPc < 32 ? kPc : 32;
#pragma unroll 1
        for (int c = part * kPc; c < (part + 1) * kPc; c += kW) {
            uint32_t a[kW];
            tmem_ldn<kW>(t_dq + lane_off + c, a);
            if (!ok) continue;
            if (slot == kDirect) {
#pragma unroll
                for (int t = 0; t < kW; t += 8) {
                    float f[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(a[t + u]) * p.scale;
                    *reinterpret_cast<uint4*>(row + c + t) = pack8(f);
                }
            } else {
#pragma unroll
                for (int t = 0; t < kW; t += 4)
                    *reinterpret_cast<float4*>(prow + c + t) =
                        make_float4(__uint_as_float(a[t]) * p.scale, __uint_as_float(a[t + 1]) * p.scale,
                                    __uint_as_float(a[t + 2]) * p.scale, __uint_as_float(a[t + 3]) * p.scale);
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

// One launch for both kinds: the dK/dV and dQ work items are independent, so
// interleaving them lets the light items of one kind fill the tail of the
// other. Explicit schedule: item blockIdx.x of the host plan. Implicit (plans
// too large for the parameter block): rank r = key block r and query block
// nb_q - 1 - r, every head, unsplit, GQA partial slot kb * nq + h.
template <int D>
__global__ void __launch_bounds__(kThreadsBwd, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const BwdParams p, const __grid_constant__ BwdSched sched, const int nq, const int nb_kv,
                       const int nb_q) {
    if (sched.n > 0) {
        BLK(0);
        const uint2 it = sched.item[blockIdx.x];
        const int h = (it.x >> 24) & 127, b = (it.x >> 16) & 255, c0 = (it.x >> 8) & 255, c1 = it.x & 255;
        if (it.x >> 31)
            attn_bwd_dq_body<D>(tm_k, tm_v, p, b, h, c0, c1, it.y);
        else
            attn_bwd_dkdv_body<D>(tm_k, tm_v, tm_q, tm_do, p, b, h, c0, c1, it.y);
        BLK(1);
        return;
    }
    const int both = min(nb_kv, nb_q);
    int rank, rem;
    bool dkdv;
    if (static_cast<int>(blockIdx.x) < 2 * nq * both) {
        rank = blockIdx.x / (2 * nq);
        rem = blockIdx.x % (2 * nq);
        dkdv = rem < nq;
        if (!dkdv) rem -= nq;
    } else {
        const int i = blockIdx.x - 2 * nq * both;
        rank = both + i / nq;
        rem = i % nq;
        dkdv = nb_kv > nb_q;
    }
    if (dkdv)
        attn_bwd_dkdv_body<D>(tm_k, tm_v, tm_q, tm_do, p, rank, rem, 0, -1,
                              p.group > 1 ? static_cast<uint32_t>(rank * nq + rem) : kDirect);
    else
        attn_bwd_dq_body<D>(tm_k, tm_v, p, nb_q - 1 - rank, rem, 0, -1, kDirect);
}

// Fixed-order sum of the partial slots -> bf16 dK / dV (blocks with partials:
// GQA group > 1 or split) and dQ (split blocks). Thread = 8 consecutive d of one
// row; the slots of (kv head, block) are its heads' chunks in (head, chunk) order.
// (A variant where the last-arriving contributor CTA summed its block's slots
// instead of this launch measured slower on B200: 75 -> 113 us at TP = 8.)
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_reduce(const float* __restrict__ dk_part,
                                                       const float* __restrict__ dv_part,
                                                       const float* __restrict__ dq_part, __nv_bfloat16* dk,
                                                       __nv_bfloat16* dv, __nv_bfloat16* dq, long long lddkv,
                                                       long long lddq, int T, int T_kv, int nq, int group, int hpi,
                                                       int nb_kv, int nb_q, const __grid_constant__ BwdSlots tb) {
    constexpr int V = D / 8;
    const int nkv = nq / group;
    const long long n_kv = static_cast<long long>(nkv) * nb_kv * BKV * V;
    const long long n_all = n_kv + static_cast<long long>(nq) * nb_q * BQ * V;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n_all;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const bool kv = i < n_kv;
        const long long j = kv ? i : i - n_kv;
        const int d8 = static_cast<int>(j % V);
        const int r = static_cast<int>((j / V) % BKV);
        const long long hb = j / (static_cast<long long>(V) * BKV);
        const int nb = kv ? nb_kv : nb_q;
        const int b = static_cast<int>(hb % nb), hh = static_cast<int>(hb / nb);
        const uint32_t base = kv ? tb.kv_base[b] : tb.q_base[b];
        const int row = b * BKV + r;
        if (base == kDirect || row >= (kv ? T_kv : T)) continue;
        const int nck = kv ? tb.kv_nck[b] : tb.q_nck[b];
        const int heads = kv ? group / hpi : 1, h0 = kv ? hh * (group / hpi) : hh;
        float sk[8] = {}, sv[8] = {};
        for (int s2 = 0; s2 < heads * nck; ++s2) {
            const long long off = ((static_cast<long long>(base) + h0 * nck + s2) * BKV + r) * D + d8 * 8;
            const float* src = kv ? dk_part : dq_part;
            const float4 a0 = *reinterpret_cast<const float4*>(src + off);
            const float4 a1 = *reinterpret_cast<const float4*>(src + off + 4);
            sk[0] += a0.x; sk[1] += a0.y; sk[2] += a0.z; sk[3] += a0.w;
            sk[4] += a1.x; sk[5] += a1.y; sk[6] += a1.z; sk[7] += a1.w;
            if (kv) {
                const float4 b0 = *reinterpret_cast<const float4*>(dv_part + off);
                const float4 b1 = *reinterpret_cast<const float4*>(dv_part + off + 4);
                sv[0] += b0.x; sv[1] += b0.y; sv[2] += b0.z; sv[3] += b0.w;
                sv[4] += b1.x; sv[5] += b1.y; sv[6] += b1.z; sv[7] += b1.w;
            }
        }
        if (kv) {
            *reinterpret_cast<uint4*>(dk + static_cast<long long>(row) * lddkv + hh * D + d8 * 8) = pack8(sk);
            *reinterpret_cast<uint4*>(dv + static_cast<long long>(row) * lddkv + hh * D + d8 * 8) = pack8(sv);
        } else {
            *reinterpret_cast<uint4*>(dq + static_cast<long long>(row) * lddq + hh * D + d8 * 8) = pack8(sk);
        }
    }
}

// Backward work plan: items and partial slots for (T, T_kv, query offset,
// heads, GQA group, SMs). Costs per item in cycles from clock64 traces of the
// kernel on B200 (tools/attn_trace.py): dK/dV 2650 per 128-query tile + 3000,
// dQ 1755 per 128-key tile + 2500. An item costlier than the average per-SM
// load is split into ceil(cost / average) chunks of its inner loop.
struct BwdPlan {
    std::vector<uint2> items;  // empty: implicit schedule
    BwdSlots slots;
    long long kv_slots = 0, q_slots = 0;
    int hpi = 1;               // q heads per dK/dV item (GQA group loop)
};

const BwdPlan* bwd_plan(int T, int T_kv, int qo, int nq, int group) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int, int>, BwdPlan> cache;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(T, T_kv, qo, nq, group);
    auto f = cache.find(key);
    if (f != cache.end()) return &f->second;
    const int nb_kv = (T_kv + BKV - 1) / BKV, nb_q = (T + BQ - 1) / BQ, nq128 = nb_q;
    if (nb_kv > kMaxBwdBlocks || nb_q > kMaxBwdBlocks) return nullptr;
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    auto n_kv = [&](int kb) { return std::max(0, nq128 - std::max(0, kb - qo)); };
    auto n_q = [&](int qb) { return std::min(qo + qb + 1, nb_kv); };
    auto cost_kv = [](int n) { return 2650.0 * n + 3000.0; };
    auto cost_q = [](int n) { return 1755.0 * n + 2500.0; };
    double W = 0.0;
    for (int b = 0; b < nb_kv; ++b) W += nq * cost_kv(n_kv(b));
    for (int b = 0; b < nb_q; ++b) W += nq * cost_q(n_q(b));
    // split threshold: a fraction of the mean per-SM load. Off by default
    // (DH_ATTN_SPLIT_FRAC unset): on B200 the TP = 8 shapes ran slower split
    // (frac 1: 75.0 -> 80.3 us, 0.5: 90.1 us) - the kernel is power-capped, so
    // the partial-slot traffic costs more than the better balance recovers.
    static const double frac = [] {
        const char* e = std::getenv("DH_ATTN_SPLIT_FRAC");
        return e ? std::atof(e) : 1e30;
    }();
    const double L = W / sms * frac;
    auto chunks = [&](double c, int n) { return n < 2 ? 1 : std::clamp(static_cast<int>(std::ceil(c / L)), 1, std::min(n, 255)); };
    BwdPlan pl;
    long long count = 0;
    std::vector<int> nck_kv(nb_kv), nck_q(nb_q);
    for (int b = 0; b < nb_kv; ++b) count += nq * (nck_kv[b] = chunks(cost_kv(n_kv(b)), n_kv(b)));
    for (int b = 0; b < nb_q; ++b) count += nq * (nck_q[b] = chunks(cost_q(n_q(b)), n_q(b)));
    const bool expl = count <= kMaxBwdItems && nq <= 127 && nq128 <= 255 && nb_kv <= 255;
    // GQA group loop: one dK/dV item per (key block, kv head) accumulates all of
    // its group's q heads in TMEM (no fp32 partial slots, no reduction) when even
    // the heaviest such item stays within the mean per-SM load (many heads per
    // GPU: TP = 1 Llama-3-8B has 8 kv heads); otherwise, with at least two kv
    // heads, the group items are split into chunks (fewer slots than per head)
    static const bool group_loop = [] {  // DH_ATTN_GROUP_LOOP=0: per-head items + reduction (A/B)
        const char* e = std::getenv("DH_ATTN_GROUP_LOOP");
        return !e || e[0] != '0';
    }();
    if (group_loop && expl && group > 1 && cost_kv(group * n_kv(0)) <= L / frac) {
        pl.hpi = group;
        std::fill(nck_kv.begin(), nck_kv.end(), 1);
    } else if (group_loop && expl && group > 1 && nq / group >= 2) {
        // group loop with the group items split into chunks of at most the mean
        // per-SM load (partial slots per chunk). B200, T = 4096: 8 q / 2 kv heads
        // 130.1 -> 114.9 us, 16 / 4: 246.0 -> 209.1 us; with a single kv head
        // (4 / 1) 72.2 -> 74.3 us, so that case keeps per-head items.
        pl.hpi = group;
        for (int b = 0; b < nb_kv; ++b) {
            const int n = n_kv(b) * group;
            nck_kv[b] = n < 2 ? 1 : std::clamp(static_cast<int>(std::ceil(cost_kv(n) / (W / sms))), 1,
                                               std::min(n_kv(b), 255));
        }
    }
    uint32_t run = 0;
    for (int b = 0; b < kMaxBwdBlocks; ++b) {
        pl.slots.kv_base[b] = pl.slots.q_base[b] = kDirect;
        pl.slots.kv_nck[b] = pl.slots.q_nck[b] = 1;
    }
    for (int b = 0; b < nb_kv; ++b) {
        const int nck = expl ? nck_kv[b] : 1;
        pl.slots.kv_nck[b] = static_cast<uint8_t>(nck);
        if ((group > 1 && pl.hpi == 1) || nck > 1) {
            pl.slots.kv_base[b] = run;
            run += nq / pl.hpi * nck;
        }
    }
    pl.kv_slots = run;
    run = 0;
    for (int b = 0; b < nb_q; ++b) {
        const int nck = expl ? nck_q[b] : 1;
        pl.slots.q_nck[b] = static_cast<uint8_t>(nck);
        if (nck > 1) {
            pl.slots.q_base[b] = run;
            run += nq * nck;
        }
    }
    pl.q_slots = run;
    if (expl) {
        struct It {
            double cost;
            uint2 it;
        };
        std::vector<It> its;
        for (int kind = 0; kind < 2; ++kind) {
            const int nb = kind ? nb_q : nb_kv;
            for (int b = 0; b < nb; ++b) {
                const int n = kind ? n_q(b) : n_kv(b);
                const int nck = kind ? pl.slots.q_nck[b] : pl.slots.kv_nck[b];
                const uint32_t base = kind ? pl.slots.q_base[b] : pl.slots.kv_base[b];
                const int hstep = kind ? 1 : pl.hpi;  // group loop: one item per kv head
                for (int h = 0; h < nq; h += hstep)
                    for (int c = 0; c < nck; ++c) {
                        const int c0 = n * c / nck, c1 = n * (c + 1) / nck;
                        const uint32_t x = (static_cast<uint32_t>(kind) << 31) | (static_cast<uint32_t>(h) << 24) |
                                           (static_cast<uint32_t>(b) << 16) | (static_cast<uint32_t>(c0) << 8) |
                                           static_cast<uint32_t>(c1);
                        const uint32_t y = base == kDirect ? kDirect : base + h / hstep * nck + c;
                        its.push_back({kind ? cost_q(c1 - c0) : cost_kv(hstep * (c1 - c0)), make_uint2(x, y)});
                    }
            }
        }
        std::stable_sort(its.begin(), its.end(), [](const It& a, const It& b) { return a.cost > b.cost; });
        for (const It& t : its) pl.items.push_back(t.it);
    }
    return &cache.emplace(key, std::move(pl)).first->second;
}

long long align4(long long n) { return (n + 3) / 4 * 4; }

template <int D>
int attn_bwd_tc_d(const void* q, const void* k, const void* v, long long ldq, long long ldkv, const void* dout,
                  long long ldo, const float* lse, const float* dvec, float* part, void* dq, void* dk, void* dv,
                  long long lddq, long long lddkv, int T, int nq, int nkv, float scale, int T_kv, int q_offset,
                  cudaStream_t s) {
    const int group = nq / nkv;
    const BwdPlan* pl = bwd_plan(T, T_kv, q_offset / BQ, nq, group);
    if (!pl) return set_error(DH_ERR_INVALID, "attn_bwd: more than 256 blocks of 128 rows");
    CUtensorMap mk, mv, mq, mdo;
    const long long qcols = static_cast<long long>(nq) * D, kvcols = static_cast<long long>(nkv) * D;
    int rc = make_tma_2d(&mk, k, kvcols, T_kv, ldkv, 64, 128);
    if (!rc) rc = make_tma_2d(&mv, v, kvcols, T_kv, ldkv, 64, 128);
    if (!rc) rc = make_tma_2d(&mq, q, qcols, T, ldq, 64, 128);
    if (!rc) rc = make_tma_2d(&mdo, dout, qcols, T, ldo, 64, 128);
    if (rc) return rc;
    constexpr int smem = KvSmem<D>::total > DqSmem<D>::total ? KvSmem<D>::total : DqSmem<D>::total;
    static bool cfg = false;
    if (!cfg) {
        DH_CUDA_CHECK(cudaFuncSetAttribute(attn_bwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cfg = true;
    }
    const int nb_kv = (T_kv + BKV - 1) / BKV, nb_q = (T + BQ - 1) / BQ;
    float* dk_part = part;
    float* dv_part = dk_part + pl->kv_slots * BKV * D;
    float* dq_part = dv_part + pl->kv_slots * BKV * D;
    BwdParams prm{static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(dout), ldq, ldo,
                  lse, dvec, dk_part, dv_part, dq_part, static_cast<__nv_bfloat16*>(dk),
                  static_cast<__nv_bfloat16*>(dv), static_cast<__nv_bfloat16*>(dq), lddkv, lddq, T,
                  group, pl->hpi, scale, scale * kLog2e, T_kv, q_offset / BQ};
    static BwdSched sched;  // host staging of the kernel parameter (launches are serialised per process)
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    sched.n = static_cast<int>(pl->items.size());
    std::copy(pl->items.begin(), pl->items.end(), sched.item);
    const int grid = sched.n > 0 ? sched.n : (nb_kv + nb_q) * nq;
    attn_bwd_tc_kernel<D><<<grid, kThreadsBwd, smem, s>>>(mk, mv, mq, mdo, prm, sched, nq, nb_kv, nb_q);
    DH_CUDA_CHECK(cudaGetLastError());
    if (pl->kv_slots + pl->q_slots > 0) {
        const long long work = (static_cast<long long>(nkv) * nb_kv + static_cast<long long>(nq) * nb_q) * BKV * (D / 8);
        const int blocks = static_cast<int>(std::min<long long>((work + 255) / 256, 148 * 8));
        attn_bwd_reduce<D><<<blocks, 256, 0, s>>>(dk_part, dv_part, dq_part, static_cast<__nv_bfloat16*>(dk),
                                                  static_cast<__nv_bfloat16*>(dv), static_cast<__nv_bfloat16*>(dq),
                                                  lddkv, lddq, T, T_kv, nq, group, pl->hpi, nb_kv, nb_q,
                                                  pl->slots);
        DH_CUDA_CHECK(cudaGetLastError());
    }
    return DH_OK;
}

}  // namespace

// Scratch of the tcgen05 backward: D_i = rowsum(dO * O) [nq * T] (16-byte
// aligned), then the plan's dK, dV and dQ partial slots.
long long attn_bwd_tc_scratch_floats(int T, int nq, int nkv, int D, int T_kv, int q_offset) {
    if (nkv <= 0 || nq % nkv || T <= 0) return 0;
    const BwdPlan* pl = bwd_plan(T, T_kv, q_offset / BQ, nq, nq / nkv);
    if (!pl) return 0;
    return align4(static_cast<long long>(nq) * T) + (2 * pl->kv_slots + pl->q_slots) * BKV * D;
}

// Host launcher for the tcgen05 backward. scratch: attn_bwd_tc_scratch_floats
// floats; dvec (its first nq * T floats) must already hold rowsum(dO * O).
int attn_bwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                const void* dout, long long ldo, const float* lse, float* scratch, void* dq, void* dk, void* dv,
                long long lddq, long long lddkv, int T, int nq, int nkv, int D, float scale, int T_kv,
                int q_offset, cudaStream_t s) {
    if (q_offset % (2 * BQ) || q_offset + T > T_kv)
        return set_error(DH_ERR_INVALID, "attn_bwd: q_offset must be a multiple of 256 and q_offset + T <= T_kv");
    float* part = scratch + align4(static_cast<long long>(nq) * T);
    if (D == 128)
        return attn_bwd_tc_d<128>(q, k, v, ldq, ldkv, dout, ldo, lse, scratch, part, dq, dk, dv, lddq, lddkv, T, nq,
                                  nkv, scale, T_kv, q_offset, s);
    if (D == 64)
        return attn_bwd_tc_d<64>(q, k, v, ldq, ldkv, dout, ldo, lse, scratch, part, dq, dk, dv, lddq, lddkv, T, nq,
                                 nkv, scale, T_kv, q_offset, s);
    return set_error(DH_ERR_INVALID, "attn: head_dim must be 64 or 128");
}

}  // namespace dh
