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
                    if (DH_ATTN_POLY && (u & 3) == 3) {
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
//
// dK/dV item — one CTA per (128-key block, q head); inner q tiles of 64:
//   S^T  = K Q^T        M128 N64  K128   A=K (smem)      B=Q (smem, K-major)
//   dP^T = V dO^T       M128 N64  K128   A=V (smem)      B=dO (smem, K-major)
//   P^T = exp(scale S^T - lse_q), dS^T = P^T (dP^T - D_q)      (thread = key row)
//   dV  += P^T dO       M128 N128 K64    A=P^T (TMEM)    B=dO (smem, MN-major)
//   dK  += dS^T Q       M128 N128 K64    A=dS^T (TMEM)   B=Q  (smem, MN-major)
//   TMEM: S^T x2 (64) | dP^T x2 (64) | dV (128) | dK (128) = 512 columns;
//   P^T / dS^T (bf16 pairs) overwrite the fp32 S^T / dP^T columns of the half
//   of the q tile they come from (columns [32 h, 32 h + 16) for half h), so the
//   elementwise results never pass through shared memory and the two halves of
//   the elementwise warps never write columns the other reads (no barrier).
// dQ item — one CTA per (128-query block, q head); inner key tiles of 64:
//   S = Q K^T, dP = dO V^T (M128 N64 K128), dS = P (dP - D)    (thread = query row)
//   dQ += dS K          M128 N128 K64    A=dS (TMEM)     B=K (smem, MN-major)
//   TMEM: S x2 | dP x2 | dQ = 384 columns.
// S/dP buffers are double-buffered: the MMA warp computes tile it+1 while the
// elementwise warps work on tile it. No atomics: dQ is produced by its own
// items and per-head dK/dV partials of a GQA group are reduced in head order
// by attn_bwd_group_reduce (attention.cu).
// ===========================================================================

namespace dh {
namespace {

constexpr int BT64 = 64;
constexpr int kHalf64 = BT64 * 64 * 2;  // 8 KB: one d-half of a 64-row tile
constexpr int kStages = 4;              // Q/dO (dK/dV items) or K/V (dQ items) ring

template <int D>
struct KvSmem {
    static constexpr int kTile = tile_bytes<D>();        // 128-row K / V tile
    static constexpr int kTile64 = BT64 * D * 2;         // 64-row tile: [D/64 d-halves][64 rows][128 B]
    static constexpr int k = 0;
    static constexpr int v = k + kTile;
    static constexpr int q = v + kTile;                  // kStages 64-row tiles
    static constexpr int dout = q + kStages * kTile64;   // kStages 64-row tiles
    static constexpr int vec = dout + kStages * kTile64; // per stage: lse[64], D[64] (raw)
    static constexpr int bars = vec + kStages * 128 * 4;
    static constexpr int total = bars + 256 + 1024;
};

constexpr int kDqStages = 6;  // K/V ring of the dQ items (Q and dO live in TMEM)
template <int D>
struct DqSmem {
    static constexpr int kTile64 = BT64 * D * 2;
    static constexpr int k = 0;                          // kDqStages 64-row tiles
    static constexpr int v = k + kDqStages * kTile64;    // kDqStages 64-row tiles
    static constexpr int bars = v + kDqStages * kTile64;
    static constexpr int total = bars + 256 + 1024;
};
static_assert(KvSmem<128>::total <= 232448 && DqSmem<128>::total <= 232448, "backward smem exceeds the sm_100 limit");

struct BwdParams {
    const __nv_bfloat16* q;     // raw rows for the TMEM-resident Q / dO of the dQ items
    const __nv_bfloat16* dout;
    long long ldq, ldo;
    const float* lse;
    const float* dvec;
    float* dk_part;
    float* dv_part;
    __nv_bfloat16* dk;
    __nv_bfloat16* dv;
    __nv_bfloat16* dq;
    long long lddkv, lddq;
    int T, group;   // T: query rows (this rank's)
    float scale, scale_log2;
    int T_kv;       // key rows
    int qo;         // query offset in 128-blocks (context parallelism), even
};

// K-major 64-row tile (one 64-wide K atom per half): k-step kk over d (0..7).
__device__ __forceinline__ uint64_t desc_k64(uint32_t base, int kk) {
    return umma_desc_sw128(base + (kk >> 2) * kHalf64 + (kk & 3) * 32, 16, 1024);
}
// MN-major 64-row tile used as B with N = d: k-step kk over rows (0..3).
__device__ __forceinline__ uint64_t desc_mn64(uint32_t base, int kk) {
    return umma_desc_sw128(base + kk * 2048, kHalf64, 1024);
}

constexpr int kThreadsBwd = 320;  // producer, MMA, 8 elementwise warps (2 per TMEM quadrant)

template <int D>
__device__ __forceinline__ void attn_bwd_dkdv_body(const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                                                   const CUtensorMap& tm_q, const CUtensorMap& tm_do,
                                                   const BwdParams& p, const int kb, const int h) {
    using KvSmem = dh::KvSmem<D>;
    constexpr int kTile = KvSmem::kTile, kTile64 = KvSmem::kTile64;
    extern __shared__ uint8_t smem_raw[];
    // offset arithmetic on the __shared__ array keeps the pointer in the shared
    // space (plain loads compile to LDS rather than generic LD)
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + KvSmem::bars);
    uint64_t* kv_full = bars + 0;
    uint64_t* q_full = bars + 1;                // [kStages] Q/dO ring
    uint64_t* q_empty = q_full + kStages;       // [kStages]
    uint64_t* s_full = q_empty + kStages;       // [2] TMEM S^T/dP^T buffers
    uint64_t* p_full = s_full + 2;              // P^T/dS^T of the current tile in TMEM
    uint64_t* acc_done = p_full + 1;            // dK/dV complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);
    float* vec = reinterpret_cast<float*>(sm + KvSmem::vec);  // [stage][lse 64 | D 64]

    const int kvh = h / p.group;
    const int nq64 = (p.T + BT64 - 1) / BT64;
    // first local q tile with a query at or after the block's first key
    const int i0 = max(0, (kb - p.qo) * BKV / BT64);
    const int n_it = max(0, nq64 - i0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        mbar_init(kv_full, 1);
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
        mbar_init(p_full, 256);
        mbar_init(acc_done, 1);
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
#pragma unroll
            for (int hh = 0; hh < D / 64; ++hh) {
                tma_load_2d(sm + KvSmem::k + hh * kHalf, &tm_k, kv_full, kvh * D + 64 * hh, kb * BKV);
                tma_load_2d(sm + KvSmem::v + hh * kHalf, &tm_v, kv_full, kvh * D + 64 * hh, kb * BKV);
            }
            for (int it = 0; it < n_it; ++it) {
                const int st = it % kStages, qi = i0 + it;
                mbar_wait(&q_empty[st], ((it / kStages) & 1) ^ 1);
                mbar_expect_tx(&q_full[st], 2 * kTile64 + (bulk_vec ? 512 : 0));
                if (bulk_vec) {
                    const long long off = static_cast<long long>(h) * p.T + qi * BT64;
                    bulk_load_1d(vec + st * 128, p.lse + off, 256, &q_full[st]);
                    bulk_load_1d(vec + st * 128 + 64, p.dvec + off, 256, &q_full[st]);
                }
                uint8_t* qd = sm + KvSmem::q + st * kTile64;
                uint8_t* od = sm + KvSmem::dout + st * kTile64;
#pragma unroll
                for (int hh = 0; hh < D / 64; ++hh) {
                    tma_load_2d(qd + hh * kHalf64, &tm_q, &q_full[st], h * D + 64 * hh, qi * BT64);
                    tma_load_2d(od + hh * kHalf64, &tm_do, &q_full[st], h * D + 64 * hh, qi * BT64);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_s = umma_idesc_bf16(128, 64, false, false);
        constexpr uint32_t id_g = umma_idesc_bf16(128, D, false, true);
        const uint32_t k_addr = smem_u32(sm + KvSmem::k), v_addr = smem_u32(sm + KvSmem::v);
        auto issue_s = [&](int it) {
            const int qs = it % kStages, sb = it & 1;  // smem ring stage, TMEM buffer
            mbar_wait(&q_full[qs], (it / kStages) & 1);
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
            const int sb = it & 1, qs = it % kStages;
            // S^T/dP^T(it+1) go into the other buffer, whose P^T/dS^T were
            // consumed by the dV/dK MMAs of it-1 (issued before, in order).
            if (it + 1 < n_it) issue_s(it + 1);
            if (lane == 0) ATR(it * 8 + 0);
            mbar_wait(p_full, it & 1);
            if (lane == 0) ATR(it * 8 + 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t q_addr = smem_u32(sm + KvSmem::q + qs * kTile64);
                const uint32_t o_addr = smem_u32(sm + KvSmem::dout + qs * kTile64);
#pragma unroll
                for (int kk = 0; kk < BT64 / 16; ++kk) {
                    // P^T / dS^T: q columns [32 h, 32 h + 32) packed at column 32 h (see below)
                    const uint32_t pc = (kk >> 1) * 32 + (kk & 1) * 8;
                    tc_mma_bf16_ts(t_dv, t_s + sb * 64 + pc, desc_mn64(o_addr, kk), id_g, (it | kk) != 0);
                    tc_mma_bf16_ts(t_dk, t_dp + sb * 64 + pc, desc_mn64(q_addr, kk), id_g, (it | kk) != 0);
                }
                tc_commit(&q_empty[qs]);
                if (it + 1 == n_it) tc_commit(acc_done);
            }
            __syncwarp();
        }
    } else {
        // 8 warps: quadrant (TMEM lanes) = warp & 3, column half = (warp - 2) >> 2
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;
        const int r = quad * 32 + lane;  // key row within the block
        const int key = kb * BKV + r;
        const int t_sm = threadIdx.x - 64;  // 0..255 among the elementwise warps
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const int key_hi = kb * BKV + BKV - 1;
        const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), m1 = f2_pack(-1.f, -1.f);
        const uint64_t nl2e = f2_pack(-kLog2e, -kLog2e);
        for (int it = 0; it < n_it; ++it) {
            const int sb = it & 1, qi = i0 + it;
            if (!bulk_vec) {
                // ragged T: stage the vectors with plain loads (s_full implies q_full)
                named_barrier(1, 256);  // previous readers of this stage are done
                if (t_sm < BT64) {
                    const int q = qi * BT64 + t_sm;
                    vec[(it % kStages) * 128 + t_sm] = q < p.T ? p.lse[static_cast<long long>(h) * p.T + q] : 0.f;
                    vec[(it % kStages) * 128 + 64 + t_sm] =
                        q < p.T ? p.dvec[static_cast<long long>(h) * p.T + q] : 0.f;
                }
                named_barrier(1, 256);
            }
            if (threadIdx.x == 64) ATR(it * 8 + 2);
            mbar_wait(&s_full[sb], (it >> 1) & 1);
            if (threadIdx.x == 64) ATR(it * 8 + 3);
            tc_fence_after();
            uint32_t a[32], b[32];
            tmem_ld32(t_s + sb * 64 + lane_off + half * 32, a);
            tmem_ld32(t_dp + sb * 64 + lane_off + half * 32, b);
            tmem_ld_wait();
            if (threadIdx.x == 64) ATR(it * 8 + 5);
            if (threadIdx.x == 64) ATR(it * 8 + 6);
            // whole tile causal-visible and in range: no per-element masking
            const int qg0 = p.qo * BQ + qi * BT64;  // global position of the tile's first query
            const bool full_tile = qg0 >= key_hi && qi * BT64 + BT64 <= p.T && key_hi < p.T_kv;
            const float2* lv = reinterpret_cast<const float2*>(vec + (it % kStages) * 128 + half * 32);
            const float2* dv2 = reinterpret_cast<const float2*>(vec + (it % kStages) * 128 + 64 + half * 32);
            uint32_t pp[16], pd[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const float2 l2 = lv[u], d2 = dv2[u];
                // x = scale_log2 * s - log2e * lse
                const uint64_t x = ffma2(f2_pack(__uint_as_float(a[2 * u]), __uint_as_float(a[2 * u + 1])), sc2,
                                         ffma2(f2_pack(l2.x, l2.y), nl2e, 0ull));
                float x0, x1;
                f2_unpack(x, x0, x1);
                float e0 = fast_exp2(x0), e1 = fast_exp2(x1);
                if (!full_tile) {
                    const int q = qi * BT64 + half * 32 + 2 * u;  // local row; global position q + qo * BQ
                    const int qg = q + p.qo * BQ;
                    if (qg < key || q >= p.T || key >= p.T_kv) e0 = 0.f;
                    if (qg + 1 < key || q + 1 >= p.T || key >= p.T_kv) e1 = 0.f;
                }
                const uint64_t e = f2_pack(e0, e1);
                // dS^T = P^T (dP^T - D)
                const uint64_t ds = ffma2(e, ffma2(f2_pack(d2.x, d2.y), m1,
                                                   f2_pack(__uint_as_float(b[2 * u]), __uint_as_float(b[2 * u + 1]))),
                                          0ull);
                float s0, s1;
                f2_unpack(ds, s0, s1);
                pp[u] = pack2(e0, e1);
                pd[u] = pack2(s0, s1);
            }
            if (threadIdx.x == 64) ATR(it * 8 + 7);
            // each half packs its bf16 pairs over the start of the fp32 columns it
            // read itself, so no half overwrites columns the other still reads
            tmem_st16(t_s + sb * 64 + lane_off + half * 32, pp);
            tmem_st16(t_dp + sb * 64 + lane_off + half * 32, pd);
            tmem_st_wait();
            tc_fence_before();
            if (threadIdx.x == 64) ATR(it * 8 + 4);
            mbar_arrive(p_full);
        }
        if (n_it > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        const bool ok = key < p.T_kv;
#pragma unroll 1
        for (int c = half * (D / 64); c < (half + 1) * (D / 64); ++c) {
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
                float* kr = p.dk_part + (static_cast<long long>(h) * p.T_kv + key) * D + c * 32;
                float* vr = p.dv_part + (static_cast<long long>(h) * p.T_kv + key) * D + c * 32;
                // keys after every query of this rank (context parallelism) get no
                // gradient; TMEM was never written for them (select, not multiply)
                const bool any = n_it > 0;
#pragma unroll
                for (int t = 0; t < 32; t += 4) {
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
__device__ __forceinline__ void attn_bwd_dq_body(const CUtensorMap& tm_q, const CUtensorMap& tm_do,
                                                 const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                                                 const BwdParams& p, const int qb, const int h) {
    using DqSmem = dh::DqSmem<D>;
    constexpr int kTile64 = DqSmem::kTile64;
    extern __shared__ uint8_t smem_raw[];
    // offset arithmetic on the __shared__ array keeps the pointer in the shared
    // space (plain loads compile to LDS rather than generic LD)
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + DqSmem::bars);
    uint64_t* q_full = bars + 0;               // Q / dO rows stored into TMEM
    uint64_t* kv_full = bars + 1;              // [kDqStages] K/V ring
    uint64_t* kv_empty = kv_full + kDqStages;  // [kDqStages]
    uint64_t* s_full = kv_empty + kDqStages;   // [2]
    uint64_t* p_full = s_full + 2;
    uint64_t* acc_done = p_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

    const int kvh = h / p.group;
    // key tiles 0 .. covering the block's last query (global position)
    const int n_it = min((p.qo * BQ + qb * BQ + BQ) / BT64, (p.T_kv + BT64 - 1) / BT64);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        mbar_init(q_full, 256);
        for (int i = 0; i < kDqStages; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
        mbar_init(p_full, 256);
        mbar_init(acc_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // S x2 | dP x2 | dQ | Q (bf16 pairs) | dO (bf16 pairs): Q and dO are the A
    // operands of every S / dP MMA, so they are read from TMEM, not shared memory
    const uint32_t t_s = tmem, t_dp = tmem + 128, t_dq = tmem + 256, t_qa = tmem + 384, t_doa = tmem + 448;

    if (warp == 0) {
        if (lane == 0) {
            for (int it = 0; it < n_it; ++it) {
                const int st = it % kDqStages;
                mbar_wait(&kv_empty[st], ((it / kDqStages) & 1) ^ 1);
                mbar_expect_tx(&kv_full[st], 2 * kTile64);
                uint8_t* kd = sm + DqSmem::k + st * kTile64;
                uint8_t* vd = sm + DqSmem::v + st * kTile64;
#pragma unroll
                for (int hh = 0; hh < D / 64; ++hh) {
                    tma_load_2d(kd + hh * kHalf64, &tm_k, &kv_full[st], kvh * D + 64 * hh, it * BT64);
                    tma_load_2d(vd + hh * kHalf64, &tm_v, &kv_full[st], kvh * D + 64 * hh, it * BT64);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_s = umma_idesc_bf16(128, 64, false, false);
        constexpr uint32_t id_g = umma_idesc_bf16(128, D, false, true);
        auto issue_s = [&](int it) {
            const int ks = it % kDqStages, sb = it & 1;
            mbar_wait(&kv_full[ks], (it / kDqStages) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t k_addr = smem_u32(sm + DqSmem::k + ks * kTile64);
                const uint32_t v_addr = smem_u32(sm + DqSmem::v + ks * kTile64);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    tc_mma_bf16_ts(t_s + sb * 64, t_qa + kk * 8, desc_k64(k_addr, kk), id_s, kk > 0);
                    tc_mma_bf16_ts(t_dp + sb * 64, t_doa + kk * 8, desc_k64(v_addr, kk), id_s, kk > 0);
                }
                tc_commit(&s_full[sb]);
            }
            __syncwarp();
        };
        mbar_wait(q_full, 0);
        tc_fence_after();
        issue_s(0);
        for (int it = 0; it < n_it; ++it) {
            const int sb = it & 1, ks = it % kDqStages;
            if (it + 1 < n_it) issue_s(it + 1);
            if (lane == 0) ATR(it * 8 + 0);
            mbar_wait(p_full, it & 1);
            if (lane == 0) ATR(it * 8 + 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t k_addr = smem_u32(sm + DqSmem::k + ks * kTile64);
#pragma unroll
                for (int kk = 0; kk < BT64 / 16; ++kk)
                    tc_mma_bf16_ts(t_dq, t_dp + sb * 64 + (kk >> 1) * 32 + (kk & 1) * 8, desc_mn64(k_addr, kk), id_g,
                                   (it | kk) != 0);
                tc_commit(&kv_empty[ks]);
                if (it + 1 == n_it) tc_commit(acc_done);
            }
            __syncwarp();
        }
    } else {
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;
        const int r = quad * 32 + lane;
        const int qrow = qb * BQ + r;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const int qc = min(qrow, p.T - 1);
        const float lse2 = p.lse[static_cast<long long>(h) * p.T + qc] * kLog2e;
        const float dd = p.dvec[static_cast<long long>(h) * p.T + qc];
        const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), nl2 = f2_pack(-lse2, -lse2);
        const uint64_t nd2 = f2_pack(-dd, -dd);
        {
            // this thread's query row of Q (half 0) or dO (half 1) into its TMEM lane:
            // row-major bf16 pairs are exactly the packed A-operand columns
            const __nv_bfloat16* src = half ? p.dout + static_cast<long long>(qc) * p.ldo + h * D
                                            : p.q + static_cast<long long>(qc) * p.ldq + h * D;
            const bool in = qrow < p.T;
#pragma unroll
            for (int c = 0; c < D / 64; ++c) {
                uint32_t w[32];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint4 x = in ? *reinterpret_cast<const uint4*>(src + c * 64 + u * 8) : make_uint4(0, 0, 0, 0);
                    w[4 * u] = x.x;
                    w[4 * u + 1] = x.y;
                    w[4 * u + 2] = x.z;
                    w[4 * u + 3] = x.w;
                }
                tmem_st32((half ? t_doa : t_qa) + lane_off + c * 32, w);
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(q_full);
        }
        for (int it = 0; it < n_it; ++it) {
            const int sb = it & 1;
            if (threadIdx.x == 64) ATR(it * 8 + 2);
            mbar_wait(&s_full[sb], (it >> 1) & 1);
            if (threadIdx.x == 64) ATR(it * 8 + 3);
            tc_fence_after();
            uint32_t a[32], b[32];
            tmem_ld32(t_s + sb * 64 + lane_off + half * 32, a);
            tmem_ld32(t_dp + sb * 64 + lane_off + half * 32, b);
            tmem_ld_wait();
            if (threadIdx.x == 64) ATR(it * 8 + 5);
            if (threadIdx.x == 64) ATR(it * 8 + 6);
            const int qg0 = (p.qo + qb) * BQ;  // global position of the block's first query
            const bool full_tile = it * BT64 + BT64 - 1 <= qg0 && it * BT64 + BT64 <= p.T_kv && qb * BQ + BQ <= p.T;
            uint32_t pd[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const uint64_t x = ffma2(f2_pack(__uint_as_float(a[2 * u]), __uint_as_float(a[2 * u + 1])), sc2, nl2);
                float x0, x1;
                f2_unpack(x, x0, x1);
                float e0 = fast_exp2(x0), e1 = fast_exp2(x1);
                if (!full_tile) {
                    const int key = it * BT64 + half * 32 + 2 * u;
                    const int qpos = qg0 + r;
                    if (key > qpos || key >= p.T_kv) e0 = 0.f;
                    if (key + 1 > qpos || key + 1 >= p.T_kv) e1 = 0.f;
                }
                const uint64_t ds =
                    ffma2(f2_pack(e0, e1), fadd2(f2_pack(__uint_as_float(b[2 * u]), __uint_as_float(b[2 * u + 1])), nd2),
                          0ull);
                float s0, s1;
                f2_unpack(ds, s0, s1);
                pd[u] = pack2(s0, s1);
            }
            if (threadIdx.x == 64) ATR(it * 8 + 7);
            tmem_st16(t_dp + sb * 64 + lane_off + half * 32, pd);  // over this half's own fp32 columns
            tmem_st_wait();
            tc_fence_before();
            if (threadIdx.x == 64) ATR(it * 8 + 4);
            mbar_arrive(p_full);
        }
        mbar_wait(acc_done, 0);
        tc_fence_after();
        const bool ok = qrow < p.T;
        __nv_bfloat16* row = p.dq + static_cast<long long>(qrow) * p.lddq + h * D;
#pragma unroll 1
        for (int c = half * (D / 64); c < (half + 1) * (D / 64); ++c) {
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

// One launch for both kinds: the dK/dV and dQ work items are independent, so
// interleaving them (rank r = r-th heaviest block of either kind, all heads)
// lets the light items of one kind fill the tail of the other. With few heads
// per GPU (high TP) two separate grids each left their longest causal block as
// an exposed critical path.
template <int D>
__global__ void __launch_bounds__(kThreadsBwd, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const __grid_constant__ CUtensorMap tm_q64, const __grid_constant__ CUtensorMap tm_do64,
                       const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_k64, const __grid_constant__ CUtensorMap tm_v64,
                       const BwdParams p, const int nq, const int nb_kv, const int nb_q) {
    // rank r: key block r (the low blocks see the most queries) and query
    // block nb_q - 1 - r (the high blocks see the most keys), every head;
    // past the shorter of the two ranges only the longer kind remains
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
        attn_bwd_dkdv_body<D>(tm_k, tm_v, tm_q64, tm_do64, p, rank, rem);
    else
        attn_bwd_dq_body<D>(tm_q, tm_do, tm_k64, tm_v64, p, nb_q - 1 - rank, rem);
}

template <int D>
int attn_bwd_tc_d(const void* q, const void* k, const void* v, long long ldq, long long ldkv, const void* dout,
                  long long ldo, const float* lse, const float* dvec, float* dk_part, float* dv_part, void* dq,
                  void* dk, void* dv, long long lddq, long long lddkv, int T, int nq, int nkv, float scale,
                  int T_kv, int q_offset, cudaStream_t s) {
    CUtensorMap mk, mv, mq64, mdo64, mq, mdo, mk64, mv64;
    const long long qcols = static_cast<long long>(nq) * D, kvcols = static_cast<long long>(nkv) * D;
    int rc = make_tma_2d(&mk, k, kvcols, T_kv, ldkv, 64, 128);
    if (!rc) rc = make_tma_2d(&mv, v, kvcols, T_kv, ldkv, 64, 128);
    if (!rc) rc = make_tma_2d(&mq64, q, qcols, T, ldq, 64, 64);
    if (!rc) rc = make_tma_2d(&mdo64, dout, qcols, T, ldo, 64, 64);
    if (!rc) rc = make_tma_2d(&mq, q, qcols, T, ldq, 64, 128);
    if (!rc) rc = make_tma_2d(&mdo, dout, qcols, T, ldo, 64, 128);
    if (!rc) rc = make_tma_2d(&mk64, k, kvcols, T_kv, ldkv, 64, 64);
    if (!rc) rc = make_tma_2d(&mv64, v, kvcols, T_kv, ldkv, 64, 64);
    if (rc) return rc;
    constexpr int smem = KvSmem<D>::total > DqSmem<D>::total ? KvSmem<D>::total : DqSmem<D>::total;
    static bool cfg = false;
    if (!cfg) {
        DH_CUDA_CHECK(cudaFuncSetAttribute(attn_bwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cfg = true;
    }
    BwdParams prm{static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(dout), ldq, ldo,
                  lse, dvec, dk_part, dv_part, static_cast<__nv_bfloat16*>(dk),
                  static_cast<__nv_bfloat16*>(dv), static_cast<__nv_bfloat16*>(dq), lddkv, lddq, T,
                  nq / nkv, scale, scale * kLog2e, T_kv, q_offset / BQ};
    const int nb_kv = (T_kv + BKV - 1) / BKV, nb_q = (T + BQ - 1) / BQ;
    attn_bwd_tc_kernel<D><<<(nb_kv + nb_q) * nq, kThreadsBwd, smem, s>>>(mk, mv, mq64, mdo64, mq, mdo, mk64, mv64,
                                                                        prm, nq, nb_kv, nb_q);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

}  // namespace

// Host launcher for the tcgen05 backward (dvec must already hold
// D_i = rowsum(dO * O)); dk_part / dv_part are used only when group > 1.
int attn_bwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                const void* dout, long long ldo, const float* lse, const float* dvec, float* dk_part,
                float* dv_part, void* dq, void* dk, void* dv, long long lddq, long long lddkv, int T,
                int nq, int nkv, int D, float scale, int T_kv, int q_offset, cudaStream_t s) {
    if (q_offset % (2 * BQ) || q_offset + T > T_kv)
        return set_error(DH_ERR_INVALID, "attn_bwd: q_offset must be a multiple of 256 and q_offset + T <= T_kv");
    if (D == 128)
        return attn_bwd_tc_d<128>(q, k, v, ldq, ldkv, dout, ldo, lse, dvec, dk_part, dv_part, dq, dk, dv, lddq,
                                  lddkv, T, nq, nkv, scale, T_kv, q_offset, s);
    if (D == 64)
        return attn_bwd_tc_d<64>(q, k, v, ldq, ldkv, dout, ldo, lse, dvec, dk_part, dv_part, dq, dk, dv, lddq,
                                 lddkv, T, nq, nkv, scale, T_kv, q_offset, s);
    return set_error(DH_ERR_INVALID, "attn: head_dim must be 64 or 128");
}

}  // namespace dh
