// MoE kernels of the moe_ep layer template (reference op_model.cpp:121-169):
//   router      (9)  logits = ln1 wr^T (fp32), softmax, top-k, renormalised weights
//   permute     (10) capacity-slot assignment in (token, k) order + row gather
//   unpermute   (15) out[t] = sum_k w[t,k] y[slot(t,k)]       (k ascending, fp32)
//   unpermute_bwd (21), permute_bwd (28), router_bwd (29)
// The expert FFNs (expert_fc1 / expert_fc2 and their grads) are per-expert
// tcgen05 GEMMs (gemm_tcgen05.cu) over the contiguous slot block of each
// expert; the all-to-alls are collectives (runtime/context.cpp).
//
// Slot layout: expert e owns slots [e*C, (e+1)*C) of a [E*C, hidden] row block,
// so expert-major blocks are contiguous and the rows bound for EP rank r
// (experts [r*E_loc, (r+1)*E_loc)) form one contiguous chunk. Empty slots are
// zero rows (their GEMM rows contribute nothing to any gradient).
//
// HBM-bound row kernels, warp per row, 16-byte vectors; every reduction has a
// fixed order and no atomics, so results are bit-reproducible (SI == sequential).
// The fp32 sums mirror oracle/layer_oracle.py MoEOracle term by term
// (__fmul_rn / __fadd_rn so no FMA contraction changes the rounding).
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "dh_capi.h"

namespace dh {
namespace {

constexpr int kMaxExperts = 64;
constexpr int kMaxTopk = 8;
constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ long long warp_id_global() {
    return (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
}
__device__ __forceinline__ long long warps_total() {
    return static_cast<long long>(gridDim.x) * blockDim.x / 32;
}

// ---------------------------------------------------------------- router fwd
// The logits GEMM (ln1 wr^T, fp32 out) runs on the tensor cores (dh_gemm); this
// kernel turns a token's logits row into softmax probabilities (in place) and
// its top-k. Thread per token; loops over kMaxExperts are unrolled so every
// per-token array stays in registers.
__global__ void __launch_bounds__(128)
    router_topk_kernel(float* __restrict__ probs, int* __restrict__ ids, float* __restrict__ wts, int tokens,
                       int E, int K) {
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= tokens) return;
    float* row = probs + t * E;
    float p[kMaxExperts];
    float mx = -INFINITY;
#pragma unroll
    for (int e = 0; e < kMaxExperts; ++e) {
        p[e] = e < E ? row[e] : -INFINITY;
        mx = fmaxf(mx, p[e]);
    }
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < kMaxExperts; ++e) {
        p[e] = e < E ? expf(p[e] - mx) : 0.f;
        sum = __fadd_rn(sum, p[e]);
    }
#pragma unroll
    for (int e = 0; e < kMaxExperts; ++e) {
        p[e] = __fdiv_rn(p[e], sum);
        if (e < E) row[e] = p[e];
    }
    // top-k by probability, ties to the lower expert id (stable argsort of -p)
    unsigned long long taken = 0ull;
    int sel[kMaxTopk];
    float top[kMaxTopk];
    float tsum = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxTopk; ++k) {
        if (k >= K) break;
        int best = -1;
        float bv = 0.f;
#pragma unroll
        for (int e = 0; e < kMaxExperts; ++e) {
            if (e >= E || (taken >> e & 1ull)) continue;
            if (best < 0 || p[e] > bv) {
                best = e;
                bv = p[e];
            }
        }
        taken |= 1ull << best;
        sel[k] = best;
        top[k] = bv;
        tsum = __fadd_rn(tsum, bv);
    }
#pragma unroll
    for (int k = 0; k < kMaxTopk; ++k) {
        if (k >= K) break;
        ids[t * K + k] = sel[k];
        wts[t * K + k] = __fdiv_rn(top[k], tsum);
    }
}

// ---------------------------------------------------------------- slot assignment
// One block per expert scans the (token, k) assignments in order; the running
// count gives each of its assignments a slot (or drops it past capacity).
constexpr int kAssignThreads = 1024;

__global__ void __launch_bounds__(kAssignThreads)
    assign_kernel(const int* __restrict__ ids, int n_assign, int C, int* __restrict__ slot,
                  int* __restrict__ slot_src) {
    __shared__ int warp_cnt[kAssignThreads / 32];
    __shared__ int base_sh;
    const int e = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) base_sh = 0;
    __syncthreads();
    for (int a0 = 0; a0 < n_assign; a0 += kAssignThreads) {
        const int a = a0 + threadIdx.x;
        const bool mine = a < n_assign && ids[a] == e;
        const unsigned ball = __ballot_sync(0xffffffffu, mine);
        if (lane == 0) warp_cnt[w] = __popc(ball);
        __syncthreads();
        int before = base_sh;
        for (int i = 0; i < w; ++i) before += warp_cnt[i];
        const int rank = before + __popc(ball & ((1u << lane) - 1u));
        if (mine) {
            if (rank < C) {
                slot[a] = e * C + rank;
                slot_src[e * C + rank] = a;
            } else {
                slot[a] = -1;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int i = 0; i < kAssignThreads / 32; ++i) tot += warp_cnt[i];
            base_sh += tot;
        }
        __syncthreads();
    }
    for (int j = min(base_sh, C) + threadIdx.x; j < C; j += kAssignThreads) slot_src[e * C + j] = -1;
}

// ---------------------------------------------------------------- permute
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    permute_kernel(const uint4* __restrict__ x, const int* __restrict__ slot_src, uint4* __restrict__ xp,
                   int n_slots, int K, int hvec) {
    const int lane = threadIdx.x & 31;
    for (long long s = warp_id_global(); s < n_slots; s += warps_total()) {
        const int a = slot_src[s];
        uint4* dst = xp + s * hvec;
        if (a < 0) {
            for (int c = lane; c < hvec; c += 32) dst[c] = make_uint4(0, 0, 0, 0);
        } else {
            const uint4* src = x + static_cast<long long>(a / K) * hvec;
            for (int c = lane; c < hvec; c += 32) dst[c] = src[c];
        }
    }
}

// ---------------------------------------------------------------- unpermute (weighted combine)
// Warp per token; KT (compile-time top-k) and two column vectors per step keep
// 2*KT independent 16-byte gathers in flight per lane.
template <int KT>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    unpermute_kernel(const uint4* __restrict__ y, const int* __restrict__ slot, const float* __restrict__ wts,
                     uint4* __restrict__ out, int tokens, int hvec) {
    const int lane = threadIdx.x & 31;
    for (long long t = warp_id_global(); t < tokens; t += warps_total()) {
        int sl[KT];
        float w[KT];
#pragma unroll
        for (int k = 0; k < KT; ++k) {
            sl[k] = slot[t * KT + k];
            w[k] = wts[t * KT + k];
        }
        // NJ 16-byte columns per lane in flight per slot row (one for top-k > 4,
        // where two would exceed the register budget)
        constexpr int NJ = KT > 4 ? 1 : 2;
        for (int c0 = lane; c0 < hvec; c0 += 32 * NJ) {
            uint4 v[KT][NJ];
#pragma unroll
            for (int k = 0; k < KT; ++k)
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    const int c = c0 + 32 * j;
                    v[k][j] = sl[k] >= 0 && c < hvec ? y[static_cast<long long>(sl[k]) * hvec + c] : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int c = c0 + 32 * j;
                if (c >= hvec) break;
                float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                for (int k = 0; k < KT; ++k) {
                    if (sl[k] < 0) continue;  // dropped: no term (not even +0 * w)
                    float f[8];
                    unpack8(v[k][j], f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], __fmul_rn(w[k], f[i]));
                }
                out[t * hvec + c] = pack8(acc);
            }
        }
    }
}

// ---------------------------------------------------------------- unpermute bwd
// dys[s] = bf16(w * dy[t]); dw[a] = <y[s], dy[t]> for the assignment a in slot s.
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    unpermute_bwd_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ y,
                         const int* __restrict__ slot_src, const float* __restrict__ wts,
                         uint4* __restrict__ dys, float* __restrict__ dw, int n_slots, int K, int hvec) {
    const int lane = threadIdx.x & 31;
    for (long long s = warp_id_global(); s < n_slots; s += warps_total()) {
        const int a = slot_src[s];
        uint4* dst = dys + s * hvec;
        if (a < 0) {
            for (int c = lane; c < hvec; c += 32) dst[c] = make_uint4(0, 0, 0, 0);
            continue;
        }
        const float w = wts[a];
        const uint4* g = dy + static_cast<long long>(a / K) * hvec;
        const uint4* yr = y + s * hvec;
        float dot = 0.f;
        for (int c = lane; c < hvec; c += 32) {
            float gv[8], yv[8], o[8];
            unpack8(g[c], gv);
            unpack8(yr[c], yv);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                o[i] = __fmul_rn(w, gv[i]);
                dot = fmaf(yv[i], gv[i], dot);
            }
            dst[c] = pack8(o);
        }
        dot = warp_sum(dot);
        if (lane == 0) dw[a] = dot;
    }
}

// ---------------------------------------------------------------- permute bwd
template <int KT>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    permute_bwd_kernel(const uint4* __restrict__ dxp, const int* __restrict__ slot, uint4* __restrict__ dx,
                       int tokens, int hvec) {
    const int lane = threadIdx.x & 31;
    for (long long t = warp_id_global(); t < tokens; t += warps_total()) {
        int sl[KT];
#pragma unroll
        for (int k = 0; k < KT; ++k) sl[k] = slot[t * KT + k];
        for (int c0 = lane; c0 < hvec; c0 += 64) {
            uint4 v[KT][2];
#pragma unroll
            for (int k = 0; k < KT; ++k)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int c = c0 + 32 * j;
                    v[k][j] = sl[k] >= 0 && c < hvec ? dxp[static_cast<long long>(sl[k]) * hvec + c] : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int c = c0 + 32 * j;
                if (c >= hvec) break;
                float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                for (int k = 0; k < KT; ++k) {
                    if (sl[k] < 0) continue;
                    float f[8];
                    unpack8(v[k][j], f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], f[i]);
                }
                dx[t * hvec + c] = pack8(acc);
            }
        }
    }
}

// ---------------------------------------------------------------- router bwd
// Per token (thread): dtop = dw/ssum - <dw, top>/ssum^2 through the
// renormalisation, dp scattered to the chosen experts, dlogits = p * (dp -
// <p, dp>) through the softmax; written as bf16, the operand of the two
// router-gradient GEMMs (dx += dlogits wr, dwr += dlogits^T ln1).
// Dropped assignments carry dw = 0.
__global__ void __launch_bounds__(128)
    router_dlogits_kernel(const float* __restrict__ probs, const int* __restrict__ ids, const int* __restrict__ slot,
                          const float* __restrict__ dw, __nv_bfloat16* __restrict__ dlogits, int ld, int tokens,
                          int E, int K) {
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= tokens) return;
    float dwk[kMaxTopk], top[kMaxTopk];
    int id[kMaxTopk];
    float ssum = 0.f, dot = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxTopk; ++k) {
        id[k] = -1;
        dwk[k] = top[k] = 0.f;
        if (k >= K) continue;
        id[k] = ids[t * K + k];
        top[k] = probs[t * E + id[k]];
        dwk[k] = slot[t * K + k] >= 0 ? dw[t * K + k] : 0.f;
        ssum = __fadd_rn(ssum, top[k]);
        dot = __fadd_rn(dot, __fmul_rn(dwk[k], top[k]));
    }
    const float ss2 = __fmul_rn(ssum, ssum);
    float dtop[kMaxTopk];
#pragma unroll
    for (int k = 0; k < kMaxTopk; ++k) dtop[k] = __fsub_rn(__fdiv_rn(dwk[k], ssum), __fdiv_rn(dot, ss2));
    // <p, dp> in expert order: only the chosen experts have dp != 0
    float pdp = 0.f;
#pragma unroll
    for (int e = 0; e < kMaxExperts; ++e) {
#pragma unroll
        for (int k = 0; k < kMaxTopk; ++k)
            if (e < E && id[k] == e) pdp = __fadd_rn(pdp, __fmul_rn(top[k], dtop[k]));
    }
    const float* pr = probs + t * E;
    __nv_bfloat16* out = dlogits + t * ld;
#pragma unroll
    for (int e = 0; e < kMaxExperts; ++e) {
        if (e >= E) break;
        float dp = 0.f;
#pragma unroll
        for (int k = 0; k < kMaxTopk; ++k)
            if (id[k] == e) dp = dtop[k];
        out[e] = __float2bfloat16_rn(__fmul_rn(pr[e], __fsub_rn(dp, pdp)));
    }
}

int row_grid(long long rows) {
    const long long b = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
    return static_cast<int>(std::max<long long>(1, std::min<long long>(b, 148LL * 16)));
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }


}  // namespace
}  // namespace dh

using namespace dh;

extern "C" {

int dh_moe_router_fwd(const void* x, const void* wr, float* probs, int* ids, float* wts, int tokens,
                      int hidden, int experts, int topk, void* stream) {
    if (experts < 2 || experts > kMaxExperts || topk < 1 || topk > kMaxTopk || topk > experts)
        return set_error(DH_ERR_INVALID, "moe_router_fwd: 2 <= experts <= 64, 1 <= topk <= min(8, experts)");
    if (tokens <= 0) return DH_OK;
    if (experts % 4) return set_error(DH_ERR_INVALID, "moe_router_fwd: experts % 4 (16-byte logits rows)");
    // logits = x wr^T on the tensor cores, fp32, into the probability buffer
    dh_gemm_args g{};
    g.a = x;
    g.lda = hidden;
    g.b = wr;
    g.ldb = hidden;
    g.d = probs;
    g.ldd = experts;
    g.d_fp32 = 1;
    g.m = tokens;
    g.n = experts;
    g.k = hidden;
    if (int rc = dh_gemm(&g, stream)) return rc;
    router_topk_kernel<<<(tokens + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(probs, ids, wts, tokens,
                                                                                           experts, topk);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

int dh_moe_assign(const int* ids, int tokens, int topk, int experts, int capacity, int* slot, int* slot_src,
                  void* stream) {
    if (experts < 1 || capacity < 1) return set_error(DH_ERR_INVALID, "moe_assign: experts, capacity >= 1");
    assign_kernel<<<experts, kAssignThreads, 0, static_cast<cudaStream_t>(stream)>>>(ids, tokens * topk, capacity,
                                                                                   slot, slot_src);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

int dh_moe_permute(const void* x, const int* slot_src, void* xp, int n_slots, int topk, int hidden, void* stream) {
    if (hidden % 8 || !al16(x) || !al16(xp)) return set_error(DH_ERR_INVALID, "moe_permute: hidden % 8, 16-B alignment");
    if (n_slots <= 0) return DH_OK;
    permute_kernel<<<row_grid(n_slots), kWarpsPerBlock * 32, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(x), slot_src, static_cast<uint4*>(xp), n_slots, topk, hidden / 8);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

int dh_moe_unpermute(const void* y, const int* slot, const float* wts, void* out, int tokens, int topk, int hidden,
                     void* stream) {
    if (hidden % 8 || topk > kMaxTopk || !al16(y) || !al16(out))
        return set_error(DH_ERR_INVALID, "moe_unpermute: hidden % 8, topk <= 8, 16-B alignment");
    if (tokens <= 0) return DH_OK;
    auto s = static_cast<cudaStream_t>(stream);
    const auto* Y = static_cast<const uint4*>(y);
    auto* O = static_cast<uint4*>(out);
    const int g = row_grid(tokens), hv = hidden / 8;
    switch (topk) {
#define DH_UNPERMUTE(KT) \
    case KT: unpermute_kernel<KT><<<g, kWarpsPerBlock * 32, 0, s>>>(Y, slot, wts, O, tokens, hv); break;
        DH_UNPERMUTE(1) DH_UNPERMUTE(2) DH_UNPERMUTE(3) DH_UNPERMUTE(4)
        DH_UNPERMUTE(5) DH_UNPERMUTE(6) DH_UNPERMUTE(7) DH_UNPERMUTE(8)
#undef DH_UNPERMUTE
        default: return set_error(DH_ERR_INVALID, "moe_unpermute: 1 <= topk <= 8");
    }
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

int dh_moe_unpermute_bwd(const void* dy, const void* y, const int* slot_src, const float* wts, void* dys, float* dw,
                         int n_slots, int topk, int hidden, void* stream) {
    if (hidden % 8 || !al16(dy) || !al16(y) || !al16(dys))
        return set_error(DH_ERR_INVALID, "moe_unpermute_bwd: hidden % 8, 16-B alignment");
    if (n_slots <= 0) return DH_OK;
    unpermute_bwd_kernel<<<row_grid(n_slots), kWarpsPerBlock * 32, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(dy), static_cast<const uint4*>(y), slot_src, wts, static_cast<uint4*>(dys), dw,
        n_slots, topk, hidden / 8);
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

int dh_moe_permute_bwd(const void* dxp, const int* slot, void* dx, int tokens, int topk, int hidden, void* stream) {
    if (hidden % 8 || topk > kMaxTopk || !al16(dxp) || !al16(dx))
        return set_error(DH_ERR_INVALID, "moe_permute_bwd: hidden % 8, topk <= 8, 16-B alignment");
    if (tokens <= 0) return DH_OK;
    auto s = static_cast<cudaStream_t>(stream);
    const auto* X = static_cast<const uint4*>(dxp);
    auto* O = static_cast<uint4*>(dx);
    const int g = row_grid(tokens), hv = hidden / 8;
    switch (topk) {
#define DH_PERMUTE_BWD(KT) \
    case KT: permute_bwd_kernel<KT><<<g, kWarpsPerBlock * 32, 0, s>>>(X, slot, O, tokens, hv); break;
        DH_PERMUTE_BWD(1) DH_PERMUTE_BWD(2) DH_PERMUTE_BWD(3) DH_PERMUTE_BWD(4)
        DH_PERMUTE_BWD(5) DH_PERMUTE_BWD(6) DH_PERMUTE_BWD(7) DH_PERMUTE_BWD(8)
#undef DH_PERMUTE_BWD
        default: return set_error(DH_ERR_INVALID, "moe_permute_bwd: 1 <= topk <= 8");
    }
    DH_CUDA_CHECK(cudaGetLastError());
    return DH_OK;
}

long long dh_moe_router_bwd_scratch_floats(int tokens, int hidden, int experts) {
    (void)hidden;
    return static_cast<long long>(tokens) * ((experts + 7) / 8 * 8) / 2 + 64;  // bf16 dlogits [T, E] (16-B rows)
}

int dh_moe_router_bwd(const float* probs, const int* ids, const int* slot, const float* dw, const void* x,
                      const void* wr, const void* dx_in, void* dx_out, float* dwr, float* scratch, int tokens,
                      int hidden, int experts, int topk, void* stream) {
    if (experts < 2 || experts > kMaxExperts || topk < 1 || topk > kMaxTopk)
        return set_error(DH_ERR_INVALID, "moe_router_bwd: 2 <= experts <= 64, 1 <= topk <= 8");
    if (tokens <= 0) return DH_OK;
    const int ld = (experts + 7) / 8 * 8;  // row pitch of the bf16 dlogits: a TMA-legal 16-byte multiple
    auto s = static_cast<cudaStream_t>(stream);
    auto* dl = reinterpret_cast<__nv_bfloat16*>(scratch);
    router_dlogits_kernel<<<(tokens + 127) / 128, 128, 0, s>>>(probs, ids, slot, dw, dl, ld, tokens, experts, topk);
    DH_CUDA_CHECK(cudaGetLastError());
    if (dx_out != dx_in)
        DH_CUDA_CHECK(cudaMemcpyAsync(dx_out, dx_in, static_cast<size_t>(tokens) * hidden * 2,
                                      cudaMemcpyDeviceToDevice, s));
    // dx += dlogits wr   (K = experts)
    dh_gemm_args g{};
    g.a = dl;
    g.lda = ld;
    g.b = wr;
    g.ldb = hidden;
    g.b_mn = 1;
    g.d = dx_out;
    g.ldd = hidden;
    g.m = tokens;
    g.n = hidden;
    g.k = experts;
    g.accumulate = 1;
    if (int rc = dh_gemm(&g, stream)) return rc;
    // dwr += dlogits^T x   (fp32 gradient, K = tokens)
    dh_gemm_args w{};
    w.a = dl;
    w.lda = ld;
    w.a_mn = 1;
    w.b = x;
    w.ldb = hidden;
    w.b_mn = 1;
    w.d = dwr;
    w.ldd = hidden;
    w.d_fp32 = 1;
    w.m = experts;
    w.n = hidden;
    w.k = tokens;
    w.accumulate = 1;
    return dh_gemm(&w, stream);
}

}  // extern "C"
