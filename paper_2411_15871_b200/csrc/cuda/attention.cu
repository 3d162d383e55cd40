// Causal GQA flash attention front end: the attn / attn_bwd nodes' C ABI
// (dh_attn_fwd / dh_attn_bwd) over the tcgen05 / TMEM / TMA kernels of
// attention_tc.cu, for head_dim 64 and 128, plus the backward's two small
// helpers: rowsum(dO * O) and the fixed-order GQA group reduction.
//
// Determinism: no atomics anywhere. The backward runs planned dK/dV items (per
// (kv block, q head[, q-tile chunk])) and dQ items (per (q block, q head[,
// key-tile chunk])); partial slots (GQA groups, split items) are summed in a
// fixed order, so the interleaved SI schedule reproduces the sequential numbers
// bit for bit.
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

}  // namespace

int attn_fwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv, void* o,
                long long ldo, float* lse, int T, int nq, int nkv, int D, float scale, float* scratch,
                long long scratch_floats, int T_kv, int q_offset, cudaStream_t s);
long long attn_fwd_tc_scratch_floats(int T, int nq, int D, int T_kv, int q_offset);
int attn_bwd_tc(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
                const void* dout, long long ldo, const float* lse, float* scratch, void* dq, void* dk, void* dv,
                long long lddq, long long lddkv, int T, int nq, int nkv, int D, float scale, int T_kv,
                int q_offset, cudaStream_t s);
long long attn_bwd_tc_scratch_floats(int T, int nq, int nkv, int D, int T_kv, int q_offset);

}  // namespace dh

namespace {

template <int D>
int launch_bwd(const void* q, const void* k, const void* v, long long ldq, long long ldkv,
               const void* o, long long ldo, const float* lse, const void* dout, void* dq, void* dk,
               void* dv, long long lddq, long long lddkv, float* scratch, int T, int nq, int nkv,
               float scale, int T_kv, int q_offset, cudaStream_t s) {
    using namespace dh;
    float* dvec = scratch;
    if (ldo % 8 || (reinterpret_cast<uintptr_t>(o) & 15) || (reinterpret_cast<uintptr_t>(dout) & 15))
        return set_error(DH_ERR_INVALID, "attn_bwd: O / dO need 16-byte aligned rows (ldo % 8 == 0)");
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (lddq % 8 || lddkv % 8 || !al16(dq) || !al16(dk) || !al16(dv) || !al16(scratch))
        return set_error(DH_ERR_INVALID, "attn_bwd: dq / dk / dv / scratch need 16-byte aligned rows");
    attn_bwd_dot_kernel<D><<<static_cast<int>((static_cast<long long>(T) * nq * (D / 8) + 255) / 256), 256, 0, s>>>(
        static_cast<const bf16*>(o), ldo, static_cast<const bf16*>(dout), dvec, T, nq);
    DH_CUDA_CHECK(cudaGetLastError());
    // tcgen05/TMEM kernel (attention_tc.cu): planned dK/dV + dQ items in one
    // launch, then the fixed-order reduction of any partial slots
    return attn_bwd_tc(q, k, v, ldq, ldkv, dout, ldo, lse, scratch, dq, dk, dv, lddq, lddkv, T, nq, nkv, D, scale,
                       T_kv, q_offset, s);
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

extern "C" long long dh_attn_bwd_scratch_floats_ex(int tokens, int n_q_heads, int n_kv_heads, int head_dim,
                                                   int tokens_kv, int q_offset) {
    if ((head_dim != 128 && head_dim != 64) || tokens <= 0 || n_q_heads <= 0) return 0;
    return dh::attn_bwd_tc_scratch_floats(tokens, n_q_heads, n_kv_heads, head_dim, tokens_kv, q_offset);
}

// Without the GQA shape or query offset: enough for any n_kv_heads at offset 0
// (a GQA group > 1 gives every key block partial slots).
extern "C" long long dh_attn_bwd_scratch_floats(int tokens, int n_q_heads, int head_dim, int tokens_kv) {
    return std::max(dh_attn_bwd_scratch_floats_ex(tokens, n_q_heads, n_q_heads, head_dim, tokens_kv, 0),
                    dh_attn_bwd_scratch_floats_ex(tokens, n_q_heads, 1, head_dim, tokens_kv, 0));
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
