// Causal GQA flash attention front end: the attn / attn_bwd nodes' C ABI
// (dh_attn_fwd / dh_attn_bwd) over the tcgen05 / TMEM / TMA kernels of
// attention_tc.cu, for head_dim 64 and 128, plus the backward's two small
// helpers: rowsum(dO * O) and the fixed-order GQA group reduction.
//
// Determinism: no atomics anywhere. The backward runs dK/dV items (one CTA per
// (kv block, q head); fp32 per-head partials reduced over the GQA group in
// head order) and dQ items (one CTA per (q block, q head)), so the interleaved
// SI schedule reproduces the sequential numbers bit for bit.
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

// ------------------------------------------------------------------ backward helpers

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

}  // namespace

int attn_fwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv, void* o,
                long long ldo, float* lse, int T, int nq, int nkv, int D, float scale, float* scratch,
                long long scratch_floats, int T_kv, int q_offset, cudaStream_t s);
long long attn_fwd_tc_scratch_floats(int T, int nq, int D, int T_kv, int q_offset);
int attn_bwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                const void* dout, long long ldo, const float* lse, const float* dvec, float* dk_part,
                float* dv_part, void* dq, void* dk, void* dv, long long lddq, long long lddkv, int T,
                int nq, int nkv, int D, float scale, int T_kv, int q_offset, cudaStream_t s);

}  // namespace dh

namespace {

template <int D>
int launch_bwd(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
               const void* o, long long ldo, const float* lse, const void* dout, void* dq, void* dk,
               void* dv, long long lddq, long long lddkv, float* scratch, int T, int nq, int nkv,
               float scale, int T_kv, int q_offset, cudaStream_t s) {
    using namespace dh;
    const int group = nq / nkv;
    float* dvec = scratch;
    float* dk_part = scratch + static_cast<long long>(nq) * T;
    float* dv_part = dk_part + static_cast<long long>(nq) * T_kv * D;
    if (ldo % 8 || (reinterpret_cast<uintptr_t>(o) & 15) || (reinterpret_cast<uintptr_t>(dout) & 15))
        return set_error(DH_ERR_INVALID, "attn_bwd: O / dO need 16-byte aligned rows (ldo % 8 == 0)");
    attn_bwd_dot_kernel<D><<<static_cast<int>((static_cast<long long>(T) * nq * (D / 8) + 255) / 256), 256, 0, s>>>(
        static_cast<const bf16*>(o), ldo, static_cast<const bf16*>(dout), dvec, T, nq);
    DH_CUDA_CHECK(cudaGetLastError());
    // tcgen05/TMEM kernel (attention_tc.cu): dK/dV items + dQ items in one launch
    const int rc = attn_bwd_tc(q, k, v, ldq, ldkv, dout, ldo, lse, dvec, dk_part, dv_part, dq, dk, dv, lddq, lddkv,
                               T, nq, nkv, D, scale, T_kv, q_offset, s);
    if (rc != DH_OK) return rc;
    if (group > 1) {  // sum the GQA group's per-head dK/dV partials in head order
        const bool vec = (reinterpret_cast<uintptr_t>(dk_part) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(dv_part) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(dk) & 15) == 0 && (reinterpret_cast<uintptr_t>(dv) & 15) == 0 &&
                         lddkv % 8 == 0;
        const long long total = static_cast<long long>(nkv) * T_kv * (vec ? D / 8 : D);
        const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
        if (vec)
            attn_bwd_group_reduce<true><<<blocks, 256, 0, s>>>(dk_part, dv_part, static_cast<bf16*>(dk),
                                                               static_cast<bf16*>(dv), lddkv, T_kv, nkv, group, D);
        else
            attn_bwd_group_reduce<false><<<blocks, 256, 0, s>>>(dk_part, dv_part, static_cast<bf16*>(dk),
                                                                static_cast<bf16*>(dv), lddkv, T_kv, nkv, group, D);
        DH_CUDA_CHECK(cudaGetLastError());
    }
    return DH_OK;
}

}  // namespace

extern "C" long long dh_attn_fwd_scratch_floats_ex(int tokens, int n_q_heads, int n_kv_heads, int head_dim,
                                                   int tokens_kv, int q_offset) {
    (void)n_kv_heads;
    if ((head_dim != 128 && head_dim != 64) || tokens <= 0 || n_q_heads <= 0) return 0;
    return dh::attn_fwd_tc_scratch_floats(tokens, n_q_heads, head_dim, tokens_kv, q_offset);
}

extern "C" long long dh_attn_fwd_scratch_floats(int tokens, int n_q_heads, int n_kv_heads, int head_dim) {
    return dh_attn_fwd_scratch_floats_ex(tokens, n_q_heads, n_kv_heads, head_dim, tokens, 0);
}

extern "C" long long dh_attn_bwd_scratch_floats(int tokens, int n_q_heads, int head_dim, int tokens_kv) {
    return static_cast<long long>(n_q_heads) * (tokens + 2LL * tokens_kv * head_dim);
}

extern "C" int dh_attn_fwd_ex(const void* q, const void* k, const void* v, long long ldq, long long ldkv, void* o,
                              long long ldo, float* lse, float* scratch, long long scratch_floats, int tokens,
                              int tokens_kv, int q_offset, int n_q_heads, int n_kv_heads, int head_dim, float scale,
                              void* stream) {
    if (n_kv_heads <= 0 || n_q_heads % n_kv_heads)
        return dh::set_error(DH_ERR_INVALID, "attn: n_q_heads must be a multiple of n_kv_heads");
    if (tokens <= 0) return DH_OK;
    // tcgen05/TMEM kernel (attention_tc.cu) for head_dim 64 and 128
    return dh::attn_fwd_tc(q, k, v, ldq, ldkv, o, ldo, lse, tokens, n_q_heads, n_kv_heads, head_dim, scale,
                           scratch, scratch_floats, tokens_kv, q_offset, static_cast<cudaStream_t>(stream));
}

extern "C" int dh_attn_fwd(const void* q, const void* k, const void* v, long long ldq,
                           long long ldkv, void* o, long long ldo, float* lse, float* scratch,
                           long long scratch_floats, int tokens, int n_q_heads, int n_kv_heads,
                           int head_dim, float scale, void* stream) {
    return dh_attn_fwd_ex(q, k, v, ldq, ldkv, o, ldo, lse, scratch, scratch_floats, tokens, tokens, 0, n_q_heads,
                          n_kv_heads, head_dim, scale, stream);
}

extern "C" int dh_attn_bwd_ex(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                              const void* o, long long ldo, const float* lse, const void* dout, void* dq, void* dk,
                              void* dv, long long lddq, long long lddkv, float* scratch, int tokens, int tokens_kv,
                              int q_offset, int n_q_heads, int n_kv_heads, int head_dim, float scale, void* stream) {
    if (n_kv_heads <= 0 || n_q_heads % n_kv_heads)
        return dh::set_error(DH_ERR_INVALID, "attn: n_q_heads must be a multiple of n_kv_heads");
    if (tokens <= 0) return DH_OK;
    auto s = static_cast<cudaStream_t>(stream);
    if (head_dim == 128)
        return launch_bwd<128>(q, k, v, ldq, ldkv, o, ldo, lse, dout, dq, dk, dv, lddq, lddkv, scratch, tokens,
                               n_q_heads, n_kv_heads, scale, tokens_kv, q_offset, s);
    if (head_dim == 64)
        return launch_bwd<64>(q, k, v, ldq, ldkv, o, ldo, lse, dout, dq, dk, dv, lddq, lddkv, scratch, tokens,
                              n_q_heads, n_kv_heads, scale, tokens_kv, q_offset, s);
    return dh::set_error(DH_ERR_INVALID, "attn: head_dim must be 64 or 128");
}

extern "C" int dh_attn_bwd(const void* q, const void* k, const void* v, long long ldq,
                           long long ldkv, const void* o, long long ldo, const float* lse,
                           const void* dout, void* dq, void* dk, void* dv, long long lddq,
                           long long lddkv, float* scratch, int tokens, int n_q_heads,
                           int n_kv_heads, int head_dim, float scale, void* stream) {
    return dh_attn_bwd_ex(q, k, v, ldq, ldkv, o, ldo, lse, dout, dq, dk, dv, lddq, lddkv, scratch, tokens, tokens, 0,
                          n_q_heads, n_kv_heads, head_dim, scale, stream);
}
