// Causal GQA flash attention, forward and backward (the attn / attn_bwd nodes).
//
// Round-1 implementation: FlashAttention-2 structure on warp-level
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate) with cp.async double-buffered,
// XOR-swizzled shared-memory tiles (conflict-free ldmatrix). Attention is ~8%
// of the layer's FLOPs at the north-star shape; the tcgen05/TMEM version is
// the planned replacement.
//
// Determinism: no atomics anywhere. The backward runs a dK/dV pass (one CTA
// per (kv block, q head), fp32 per-head partials reduced over the GQA group in
// fixed order) and a separate dQ pass (one CTA per (q block, q head)), so the
// interleaved SI schedule reproduces the sequential numbers bit for bit.
//
// Layout: q/k/v/o rows are tokens, columns head-major (head h occupies
// [h*D, (h+1)*D)), arbitrary row pitch. lse is fp32 [n_q_heads, tokens],
// natural-log units: lse = log sum_j exp(scale * q.k_j).
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "dh_capi.h"

namespace dh {
namespace {

using bf16 = __nv_bfloat16;
constexpr int BT = 64;  // tokens per tile (both q and kv)
constexpr int kThr = 128;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Swizzled [BT][D] tile: 16-byte chunk c of row r lives at chunk c ^ (r & 7).
template <int D>
__device__ __forceinline__ bf16* tile_at(bf16* base, int r, int chunk) {
    return base + r * D + ((chunk ^ (r & 7)) << 3);
}

template <int D>
__device__ __forceinline__ void load_tile(bf16* s, const bf16* g, long long ld, int r0, int T) {
    constexpr int CH = D / 8;
    for (int idx = threadIdx.x; idx < BT * CH; idx += kThr) {
        const int r = idx / CH, c = idx % CH;
        const int gr = r0 + r;
        const bool ok = gr < T;
        cp_async16(tile_at<D>(s, r, c), g + static_cast<long long>(ok ? gr : 0) * ld + c * 8, ok);
    }
}

// A fragments (16 rows starting at row0, all D columns) of a swizzled tile.
template <int D>
__device__ __forceinline__ void load_a_frags(uint32_t (&f)[D / 16][4], bf16* s, int row0) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) ldsm_x4(f[kk], tile_at<D>(s, row0 + (lane & 15), kk * 2 + (lane >> 4)));
}

// acc[16 x 64] += A(16 x D, register frags) * T^T where T is a [64][D] tile
// (i.e. scores against the 64 rows of T).
template <int D>
__device__ __forceinline__ void mma_rows_x_tileT(float (&acc)[8][4], const uint32_t (&a)[D / 16][4],
                                                 bf16* t) {
    const int lane = threadIdx.x & 31;
    const int j4 = lane >> 3, r = lane & 7;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
        for (int np = 0; np < 4; ++np) {
            uint32_t b[4];
            ldsm_x4(b, tile_at<D>(t, np * 16 + (j4 >> 1) * 8 + r, kk * 2 + (j4 & 1)));
            mma16816(acc[2 * np], a[kk], b[0], b[1]);
            mma16816(acc[2 * np + 1], a[kk], b[2], b[3]);
        }
    }
}

// acc[16 x D] += P(16 x 64, fp32 accum layout) * T where T is a [64][D] tile.
template <int D>
__device__ __forceinline__ void mma_p_x_tile(float (&acc)[D / 8][4], const float (&p)[8][4], bf16* t) {
    const int lane = threadIdx.x & 31;
    const int j4 = lane >> 3, r = lane & 7;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        uint32_t a[4];
        a[0] = pack2(p[2 * kk][0], p[2 * kk][1]);
        a[1] = pack2(p[2 * kk][2], p[2 * kk][3]);
        a[2] = pack2(p[2 * kk + 1][0], p[2 * kk + 1][1]);
        a[3] = pack2(p[2 * kk + 1][2], p[2 * kk + 1][3]);
#pragma unroll
        for (int dn = 0; dn < D / 16; ++dn) {
            uint32_t b[4];
            ldsm_x4_t(b, tile_at<D>(t, kk * 16 + (j4 & 1) * 8 + r, dn * 2 + (j4 >> 1)));
            mma16816(acc[2 * dn], a, b[0], b[1]);
            mma16816(acc[2 * dn + 1], a, b[2], b[3]);
        }
    }
}

// ------------------------------------------------------------------ forward

template <int D>
__global__ void __launch_bounds__(kThr) attn_fwd_kernel(const bf16* __restrict__ q,
                                                        const bf16* __restrict__ k,
                                                        const bf16* __restrict__ v, long long ldq,
                                                        long long ldkv, bf16* __restrict__ o,
                                                        long long ldo, float* __restrict__ lse,
                                                        int T, int group, float scale_log2) {
    extern __shared__ __align__(128) uint8_t smem[];
    bf16* sQ = reinterpret_cast<bf16*>(smem);
    bf16* sK = sQ + BT * D;      // 2 buffers
    bf16* sV = sK + 2 * BT * D;  // 2 buffers

    const int qb = gridDim.x - 1 - blockIdx.x;  // heaviest (longest causal row) first
    const int h = blockIdx.y;
    const int kvh = h / group;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tq = lane & 3;
    const bf16* qh = q + h * D;
    const bf16* kh = k + kvh * D;
    const bf16* vh = v + kvh * D;
    const int n_kv = qb + 1;

    load_tile<D>(sQ, qh, ldq, qb * BT, T);
    load_tile<D>(sK, kh, ldkv, 0, T);
    load_tile<D>(sV, vh, ldkv, 0, T);
    cp_commit();

    uint32_t qf[D / 16][4];
    float acc[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    const int qrow0 = qb * BT + warp * 16 + g;  // this thread's rows: qrow0, qrow0 + 8

    for (int j = 0; j < n_kv; ++j) {
        const int buf = j & 1;
        if (j + 1 < n_kv) {
            load_tile<D>(sK + (buf ^ 1) * BT * D, kh, ldkv, (j + 1) * BT, T);
            load_tile<D>(sV + (buf ^ 1) * BT * D, vh, ldkv, (j + 1) * BT, T);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (j == 0) load_a_frags<D>(qf, sQ, warp * 16);

        float s[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
        mma_rows_x_tileT<D>(s, qf, sK + buf * BT * D);

        const bool diag = j == qb;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = j * BT + nt * 8 + 2 * tq + (e & 1);
                const int qr = qrow0 + (e >> 1) * 8;
                float x = s[nt][e] * scale_log2;
                if ((diag && key > qr) || key >= T) x = -INFINITY;
                s[nt][e] = x;
            }
        }
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            float mx = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) mx = fmaxf(mx, fmaxf(s[nt][2 * hr], s[nt][2 * hr + 1]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float m_new = fmaxf(m_run[hr], mx);
            const float base = m_new == -INFINITY ? 0.f : m_new;
            const float corr = exp2f(m_run[hr] - base);
            m_run[hr] = m_new;
            float rs = 0.f;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                s[nt][2 * hr] = exp2f(s[nt][2 * hr] - base);
                s[nt][2 * hr + 1] = exp2f(s[nt][2 * hr + 1] - base);
                rs += s[nt][2 * hr] + s[nt][2 * hr + 1];
            }
            l_run[hr] = l_run[hr] * corr + rs;
#pragma unroll
            for (int dn = 0; dn < D / 8; ++dn) {
                acc[dn][2 * hr] *= corr;
                acc[dn][2 * hr + 1] *= corr;
            }
        }
        mma_p_x_tile<D>(acc, s, sV + buf * BT * D);
        __syncthreads();
    }

#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        float l = l_run[hr];
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        const int qr = qrow0 + hr * 8;
        const float inv = l > 0.f ? 1.f / l : 0.f;
        if (qr < T) {
            bf16* orow = o + static_cast<long long>(qr) * ldo + h * D;
#pragma unroll
            for (int dn = 0; dn < D / 8; ++dn) {
                *reinterpret_cast<uint32_t*>(orow + dn * 8 + 2 * tq) =
                    pack2(acc[dn][2 * hr] * inv, acc[dn][2 * hr + 1] * inv);
            }
            if (tq == 0) {
                lse[static_cast<long long>(h) * T + qr] = (m_run[hr] + log2f(l)) * (1.f / kLog2e);
            }
        }
    }
}

// ------------------------------------------------------------------ backward

// Di = sum_d dO[i, d] * O[i, d], fp32 [heads, T]; one warp per (token, head).
template <int D>
__global__ void attn_bwd_dot_kernel(const bf16* __restrict__ o, long long ldo,
                                    const bf16* __restrict__ dout, float* __restrict__ dvec, int T,
                                    int heads) {
    // D/8 lanes per (token, head) row, one 16-byte vector of O and dO each
    constexpr int kL = D / 8;
    const long long gid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long row = gid / kL;
    const int sub = static_cast<int>(gid % kL);
    const bool ok = row < static_cast<long long>(T) * heads;
    float sum = 0.f;
    int t = 0, h = 0;
    if (ok) {
        t = static_cast<int>(row / heads);
        h = static_cast<int>(row % heads);
        float a[8], b[8];
        unpack8(*reinterpret_cast<const uint4*>(o + static_cast<long long>(t) * ldo + h * D + sub * 8), a);
        unpack8(*reinterpret_cast<const uint4*>(dout + static_cast<long long>(t) * ldo + h * D + sub * 8), b);
#pragma unroll
        for (int i = 0; i < 8; ++i) sum += a[i] * b[i];
    }
#pragma unroll
    for (int off = kL / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (ok && sub == 0) dvec[static_cast<long long>(h) * T + t] = sum;
}

// dK, dV for one kv block and one q head: warp w owns keys [16w, 16w+16).
//   S^T = K Q^T; P^T = exp(scale*S^T - lse); dP^T = V dO^T; dS^T = P^T (dP^T - Di)
//   dV += P^T dO;  dK += scale * dS^T Q
template <int D>
__global__ void __launch_bounds__(kThr) attn_bwd_dkdv_kernel(
    const bf16* __restrict__ q, const bf16* __restrict__ k, const bf16* __restrict__ v,
    long long ldq, long long ldkv, const bf16* __restrict__ dout, long long ldo,
    const float* __restrict__ lse, const float* __restrict__ dvec, float* __restrict__ dk_part,
    float* __restrict__ dv_part, bf16* __restrict__ dk_out, bf16* __restrict__ dv_out,
    long long lddkv, int T, int group, float scale) {
    extern __shared__ __align__(128) uint8_t smem[];
    bf16* sK = reinterpret_cast<bf16*>(smem);
    bf16* sV = sK + BT * D;
    bf16* sQ = sV + BT * D;          // 2 buffers
    bf16* sO = sQ + 2 * BT * D;      // dO, 2 buffers
    float* sL = reinterpret_cast<float*>(sO + 2 * BT * D);  // lse, 2 x BT
    float* sDv = sL + 2 * BT;                                // Di, 2 x BT

    const int nkb = gridDim.x;
    const int kb = nkb - 1 - blockIdx.x;  // keys near the start see the most q blocks
    const int h = blockIdx.y;
    const int kvh = h / group;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tq = lane & 3;
    const bf16* qh = q + h * D;
    const bf16* doh = dout + h * D;
    const float* lh = lse + static_cast<long long>(h) * T;
    const float* dh_ = dvec + static_cast<long long>(h) * T;
    const int nqb = (T + BT - 1) / BT;
    const float scale_log2 = scale * kLog2e;

    load_tile<D>(sK, k + kvh * D, ldkv, kb * BT, T);
    load_tile<D>(sV, v + kvh * D, ldkv, kb * BT, T);
    auto load_q_side = [&](int qb, int buf) {
        load_tile<D>(sQ + buf * BT * D, qh, ldq, qb * BT, T);
        load_tile<D>(sO + buf * BT * D, doh, ldo, qb * BT, T);
        for (int i = threadIdx.x; i < BT; i += kThr) {
            const int t = qb * BT + i;
            sL[buf * BT + i] = t < T ? lh[t] : 0.f;
            sDv[buf * BT + i] = t < T ? dh_[t] : 0.f;
        }
    };
    load_q_side(kb, 0);
    cp_commit();

    float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
    const int key0 = kb * BT + warp * 16 + g;  // rows key0, key0 + 8

    for (int qb = kb; qb < nqb; ++qb) {
        const int buf = (qb - kb) & 1;
        if (qb + 1 < nqb) {
            load_q_side(qb + 1, buf ^ 1);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        bf16* tQ = sQ + buf * BT * D;
        bf16* tO = sO + buf * BT * D;
        const float* L = sL + buf * BT;
        const float* Dv = sDv + buf * BT;

        float p[8][4], dp[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) p[i][e] = dp[i][e] = 0.f;
        {   // K / V fragments are re-read from smem each q block to stay under 255 registers
            uint32_t f[D / 16][4];
            load_a_frags<D>(f, sK, warp * 16);
            mma_rows_x_tileT<D>(p, f, tQ);   // S^T (keys x queries)
        }
        {
            uint32_t f[D / 16][4];
            load_a_frags<D>(f, sV, warp * 16);
            mma_rows_x_tileT<D>(dp, f, tO);  // dP^T
        }
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int qi = nt * 8 + 2 * tq + (e & 1);
                const int qr = qb * BT + qi;
                const int key = key0 + (e >> 1) * 8;
                float pv = exp2f(p[nt][e] * scale_log2 - L[qi] * kLog2e);
                if (key > qr || qr >= T || key >= T) pv = 0.f;
                p[nt][e] = pv;
                dp[nt][e] = pv * (dp[nt][e] - Dv[qi]);  // dS^T
            }
        }
        mma_p_x_tile<D>(dv, p, tO);
        mma_p_x_tile<D>(dk, dp, tQ);
        __syncthreads();
    }

    // Write: fp32 per-head partials when heads share a kv head, else bf16 directly.
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int key = key0 + hr * 8;
        if (key >= T) continue;
        if (group == 1) {
            bf16* krow = dk_out + static_cast<long long>(key) * lddkv + kvh * D;
            bf16* vrow = dv_out + static_cast<long long>(key) * lddkv + kvh * D;
#pragma unroll
            for (int dn = 0; dn < D / 8; ++dn) {
                *reinterpret_cast<uint32_t*>(krow + dn * 8 + 2 * tq) =
                    pack2(dk[dn][2 * hr] * scale, dk[dn][2 * hr + 1] * scale);
                *reinterpret_cast<uint32_t*>(vrow + dn * 8 + 2 * tq) =
                    pack2(dv[dn][2 * hr], dv[dn][2 * hr + 1]);
            }
        } else {
            float* krow = dk_part + (static_cast<long long>(h) * T + key) * D;
            float* vrow = dv_part + (static_cast<long long>(h) * T + key) * D;
#pragma unroll
            for (int dn = 0; dn < D / 8; ++dn) {
                *reinterpret_cast<float2*>(krow + dn * 8 + 2 * tq) =
                    make_float2(dk[dn][2 * hr] * scale, dk[dn][2 * hr + 1] * scale);
                *reinterpret_cast<float2*>(vrow + dn * 8 + 2 * tq) =
                    make_float2(dv[dn][2 * hr], dv[dn][2 * hr + 1]);
            }
        }
    }
}

// Sum the GQA group's per-head partials in head order -> bf16 dk, dv.
// VEC: 8 consecutive d per thread (two 16-byte loads per partial, one 16-byte
// store) when the partials are 16-byte aligned; else one element per thread.
template <bool VEC>
__global__ void attn_bwd_group_reduce(const float* __restrict__ dk_part,
                                      const float* __restrict__ dv_part, bf16* __restrict__ dk,
                                      bf16* __restrict__ dv, long long lddkv, int T, int n_kv,
                                      int group, int D) {
    constexpr int W = VEC ? 8 : 1;
    const long long total = static_cast<long long>(n_kv) * T * (D / W);
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int d = static_cast<int>(i % (D / W)) * W;
        const long long rest = i / (D / W);
        const int t = static_cast<int>(rest % T);
        const int kvh = static_cast<int>(rest / T);
        float sk[W] = {}, sv[W] = {};
        for (int j = 0; j < group; ++j) {  // head order: deterministic
            const long long off = (static_cast<long long>(kvh * group + j) * T + t) * D + d;
#pragma unroll
            for (int u = 0; u < W; u += (VEC ? 4 : 1)) {
                if constexpr (VEC) {
                    const float4 kk = *reinterpret_cast<const float4*>(dk_part + off + u);
                    const float4 vv = *reinterpret_cast<const float4*>(dv_part + off + u);
                    sk[u] += kk.x; sk[u + 1] += kk.y; sk[u + 2] += kk.z; sk[u + 3] += kk.w;
                    sv[u] += vv.x; sv[u + 1] += vv.y; sv[u + 2] += vv.z; sv[u + 3] += vv.w;
                } else {
                    sk[u] += dk_part[off + u];
                    sv[u] += dv_part[off + u];
                }
            }
        }
        bf16* pk = dk + static_cast<long long>(t) * lddkv + kvh * D + d;
        bf16* pv = dv + static_cast<long long>(t) * lddkv + kvh * D + d;
        if constexpr (VEC) {
            *reinterpret_cast<uint4*>(pk) = pack8(sk);
            *reinterpret_cast<uint4*>(pv) = pack8(sv);
        } else {
            *pk = __float2bfloat16(sk[0]);
            *pv = __float2bfloat16(sv[0]);
        }
    }
}

// dQ for one q block and head: warp w owns queries [16w, 16w+16).
//   S = Q K^T; P = exp(scale*S - lse); dP = dO V^T; dS = P (dP - Di); dQ += scale * dS K
template <int D>
__global__ void __launch_bounds__(kThr) attn_bwd_dq_kernel(
    const bf16* __restrict__ q, const bf16* __restrict__ k, const bf16* __restrict__ v,
    long long ldq, long long ldkv, const bf16* __restrict__ dout, long long ldo,
    const float* __restrict__ lse, const float* __restrict__ dvec, bf16* __restrict__ dq,
    long long lddq, int T, int group, float scale) {
    extern __shared__ __align__(128) uint8_t smem[];
    bf16* sQ = reinterpret_cast<bf16*>(smem);
    bf16* sO = sQ + BT * D;
    bf16* sK = sO + BT * D;      // 2 buffers
    bf16* sV = sK + 2 * BT * D;  // 2 buffers

    const int qb = gridDim.x - 1 - blockIdx.x;
    const int h = blockIdx.y;
    const int kvh = h / group;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tq = lane & 3;
    const bf16* kh = k + kvh * D;
    const bf16* vh = v + kvh * D;
    const float scale_log2 = scale * kLog2e;

    load_tile<D>(sQ, q + h * D, ldq, qb * BT, T);
    load_tile<D>(sO, dout + h * D, ldo, qb * BT, T);
    load_tile<D>(sK, kh, ldkv, 0, T);
    load_tile<D>(sV, vh, ldkv, 0, T);
    cp_commit();

    const int qrow0 = qb * BT + warp * 16 + g;
    float lrow[2], drow[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int qr = min(qrow0 + hr * 8, T - 1);
        lrow[hr] = lse[static_cast<long long>(h) * T + qr] * kLog2e;
        drow[hr] = dvec[static_cast<long long>(h) * T + qr];
    }
    uint32_t qf[D / 16][4], of[D / 16][4];
    float acc[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

    const int n_kv = qb + 1;
    for (int j = 0; j < n_kv; ++j) {
        const int buf = j & 1;
        if (j + 1 < n_kv) {
            load_tile<D>(sK + (buf ^ 1) * BT * D, kh, ldkv, (j + 1) * BT, T);
            load_tile<D>(sV + (buf ^ 1) * BT * D, vh, ldkv, (j + 1) * BT, T);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (j == 0) {
            load_a_frags<D>(qf, sQ, warp * 16);
            load_a_frags<D>(of, sO, warp * 16);
        }
        float s[8][4], dp[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
        mma_rows_x_tileT<D>(s, qf, sK + buf * BT * D);
        mma_rows_x_tileT<D>(dp, of, sV + buf * BT * D);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = j * BT + nt * 8 + 2 * tq + (e & 1);
                const int hr = e >> 1;
                const int qr = qrow0 + hr * 8;
                float pv = exp2f(s[nt][e] * scale_log2 - lrow[hr]);
                if (key > qr || key >= T) pv = 0.f;
                s[nt][e] = pv * (dp[nt][e] - drow[hr]);  // dS
            }
        }
        mma_p_x_tile<D>(acc, s, sK + buf * BT * D);
        __syncthreads();
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int qr = qrow0 + hr * 8;
        if (qr >= T) continue;
        bf16* row = dq + static_cast<long long>(qr) * lddq + h * D;
#pragma unroll
        for (int dn = 0; dn < D / 8; ++dn) {
            *reinterpret_cast<uint32_t*>(row + dn * 8 + 2 * tq) =
                pack2(acc[dn][2 * hr] * scale, acc[dn][2 * hr + 1] * scale);
        }
    }
}

}  // namespace

int attn_fwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv, void* o,
                long long ldo, float* lse, int T, int nq, int nkv, float scale, float* scratch,
                long long scratch_floats, cudaStream_t s);
long long attn_fwd_tc_scratch_floats(int T, int nq);
int attn_bwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                const void* dout, long long ldo, const float* lse, const float* dvec, float* dk_part,
                float* dv_part, void* dq, void* dk, void* dv, long long lddq, long long lddkv, int T,
                int nq, int nkv, float scale, cudaStream_t s);

}  // namespace dh

namespace {

#define RT_TC(expr)                 \
    do {                            \
        const int rc_ = (expr);     \
        if (rc_ != DH_OK) return rc_; \
    } while (0)

template <int D>
int launch_fwd(const void* q, const void* k, const void* v, long long ldq, long long ldkv, void* o,
               long long ldo, float* lse, int T, int nq, int nkv, float scale, cudaStream_t s) {
    using namespace dh;
    const int smem = 5 * BT * D * 2;
    static bool cfg = false;
    if (!cfg) {
        DH_CUDA_CHECK(cudaFuncSetAttribute(attn_fwd_kernel<D>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cfg = true;
    }
    const dim3 grid((T + BT - 1) / BT, nq);
    attn_fwd_kernel<D><<<grid, kThr, smem, s>>>(
        static_cast<const bf16*>(q), static_cast<const bf16*>(k), static_cast<const bf16*>(v), ldq,
        ldkv, static_cast<bf16*>(o), ldo, lse, T, nq / nkv, scale * kLog2e);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

template <int D>
int launch_bwd(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
               const void* o, long long ldo, const float* lse, const void* dout, void* dq, void* dk,
               void* dv, long long lddq, long long lddkv, float* scratch, int T, int nq, int nkv,
               float scale, cudaStream_t s) {
    using namespace dh;
    const int group = nq / nkv;
    float* dvec = scratch;
    float* dk_part = scratch + static_cast<long long>(nq) * T;
    float* dv_part = dk_part + static_cast<long long>(nq) * T * D;
    if (ldo % 8 || (reinterpret_cast<uintptr_t>(o) & 15) || (reinterpret_cast<uintptr_t>(dout) & 15))
        return set_error(DH_ERR_INVALID, "attn_bwd: O / dO need 16-byte aligned rows (ldo % 8 == 0)");
    {
        attn_bwd_dot_kernel<D><<<static_cast<int>((static_cast<long long>(T) * nq * (D / 8) + 255) / 256), 256, 0, s>>>(
            static_cast<const bf16*>(o), ldo, static_cast<const bf16*>(dout), dvec, T, nq);
        DH_CUDA_CHECK(cudaGetLastError());
    }
    const int nb = (T + BT - 1) / BT;
    if constexpr (D == 128) {
        // tcgen05/TMEM kernels (attention_tc.cu): dK/dV pass + dQ pass
        RT_TC(attn_bwd_tc(q, k, v, ldq, ldkv, dout, ldo, lse, dvec, dk_part, dv_part, dq, dk, dv, lddq,
                          lddkv, T, nq, nkv, scale, s));
    } else {
        const int smem = 6 * BT * D * 2 + 4 * BT * 4;
        static bool cfg = false;
        if (!cfg) {
            DH_CUDA_CHECK(cudaFuncSetAttribute(attn_bwd_dkdv_kernel<D>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            cfg = true;
        }
        attn_bwd_dkdv_kernel<D><<<dim3(nb, nq), kThr, smem, s>>>(
            static_cast<const bf16*>(q), static_cast<const bf16*>(k), static_cast<const bf16*>(v),
            ldq, ldkv, static_cast<const bf16*>(dout), ldo, lse, dvec, dk_part, dv_part,
            static_cast<bf16*>(dk), static_cast<bf16*>(dv), lddkv, T, group, scale);
        DH_CUDA_CHECK(cudaGetLastError());
    }
    if (group > 1) {  // sum the GQA group's per-head dK/dV partials in head order
        const bool vec = (reinterpret_cast<uintptr_t>(dk_part) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(dv_part) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(dk) & 15) == 0 && (reinterpret_cast<uintptr_t>(dv) & 15) == 0 &&
                         lddkv % 8 == 0;
        const long long total = static_cast<long long>(nkv) * T * (vec ? D / 8 : D);
        const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
        if (vec)
            attn_bwd_group_reduce<true><<<blocks, 256, 0, s>>>(dk_part, dv_part, static_cast<bf16*>(dk),
                                                               static_cast<bf16*>(dv), lddkv, T, nkv, group, D);
        else
            attn_bwd_group_reduce<false><<<blocks, 256, 0, s>>>(dk_part, dv_part, static_cast<bf16*>(dk),
                                                                static_cast<bf16*>(dv), lddkv, T, nkv, group, D);
        DH_CUDA_CHECK(cudaGetLastError());
    }
    if constexpr (D != 128) {
        const int smem = 6 * BT * D * 2;
        static bool cfg = false;
        if (!cfg) {
            DH_CUDA_CHECK(cudaFuncSetAttribute(attn_bwd_dq_kernel<D>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            cfg = true;
        }
        attn_bwd_dq_kernel<D><<<dim3(nb, nq), kThr, smem, s>>>(
            static_cast<const bf16*>(q), static_cast<const bf16*>(k), static_cast<const bf16*>(v),
            ldq, ldkv, static_cast<const bf16*>(dout), ldo, lse, dvec, static_cast<bf16*>(dq), lddq,
            T, group, scale);
        DH_CUDA_CHECK(cudaGetLastError());
    }
    return DH_OK;
}

}  // namespace

extern "C" long long dh_attn_fwd_scratch_floats(int tokens, int n_q_heads, int n_kv_heads, int head_dim) {
    (void)n_kv_heads;
    if (head_dim != 128 || tokens <= 0 || n_q_heads <= 0) return 0;
    return dh::attn_fwd_tc_scratch_floats(tokens, n_q_heads);
}

extern "C" int dh_attn_fwd(const void* q, const void* k, const void* v, long long ldq,
                           long long ldkv, void* o, long long ldo, float* lse, float* scratch,
                           long long scratch_floats, int tokens, int n_q_heads, int n_kv_heads,
                           int head_dim, float scale, void* stream) {
    if (n_kv_heads <= 0 || n_q_heads % n_kv_heads)
        return dh::set_error(DH_ERR_INVALID, "attn: n_q_heads must be a multiple of n_kv_heads");
    if (tokens <= 0) return DH_OK;
    auto s = static_cast<cudaStream_t>(stream);
    // head_dim 128 (every production shape): tcgen05/TMEM kernel (attention_tc.cu)
    if (head_dim == 128)
        return dh::attn_fwd_tc(q, k, v, ldq, ldkv, o, ldo, lse, tokens, n_q_heads, n_kv_heads, scale,
                               scratch, scratch_floats, s);
    if (head_dim == 64) return launch_fwd<64>(q, k, v, ldq, ldkv, o, ldo, lse, tokens, n_q_heads, n_kv_heads, scale, s);
    return dh::set_error(DH_ERR_INVALID, "attn: head_dim must be 64 or 128");
}

extern "C" int dh_attn_bwd(const void* q, const void* k, const void* v, long long ldq,
                           long long ldkv, const void* o, long long ldo, const float* lse,
                           const void* dout, void* dq, void* dk, void* dv, long long lddq,
                           long long lddkv, float* scratch, int tokens, int n_q_heads,
                           int n_kv_heads, int head_dim, float scale, void* stream) {
    if (n_kv_heads <= 0 || n_q_heads % n_kv_heads)
        return dh::set_error(DH_ERR_INVALID, "attn: n_q_heads must be a multiple of n_kv_heads");
    if (tokens <= 0) return DH_OK;
    auto s = static_cast<cudaStream_t>(stream);
    if (head_dim == 128)
        return launch_bwd<128>(q, k, v, ldq, ldkv, o, ldo, lse, dout, dq, dk, dv, lddq, lddkv, scratch,
                               tokens, n_q_heads, n_kv_heads, scale, s);
    if (head_dim == 64)
        return launch_bwd<64>(q, k, v, ldq, ldkv, o, ldo, lse, dout, dq, dk, dv, lddq, lddkv, scratch,
                              tokens, n_q_heads, n_kv_heads, scale, s);
    return dh::set_error(DH_ERR_INVALID, "attn: head_dim must be 64 or 128");
}
