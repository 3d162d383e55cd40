// MoE layer nodes (moe_ep template, reference op_model.cpp:121-169) on one EP
// rank. Attention, norms and residuals are the dense launchers (same kernels,
// renumbered ids); the MLP block becomes
//   fwd  9 router  10 permute  11 a2a_dispatch  12 expert_fc1(+SwiGLU)  13 expert_fc2
//        14 a2a_combine  15 unpermute  (16 bda1 = dense 14)
//   bwd (20 bda1_bwd = dense 20)  21 unpermute_bwd  22 a2a_combine_bwd
//        23 expert_fc2_dgrad(+SwiGLU bwd)  24 expert_fc2_wgrad  25 expert_fc1_dgrad
//        26 expert_fc1_wgrad  27 a2a_dispatch_bwd  28 permute_bwd  29 router_bwd
//        (30..40 = dense 28..38)
// Buffers (model.cpp): the source side is [experts][capacity][hidden] (the
// rows for EP rank r are one contiguous chunk), the expert side after the
// dispatch all-to-all is [e_loc][ep][capacity][hidden], so each local expert's
// rows are contiguous and its FFN is one GEMM of ep * capacity rows. With
// ep == 1 the all-to-all nodes do not exist and both sides are the same buffer.
#include <cuda_bf16.h>

#include "runtime.hpp"

namespace dh {

int moe_capacity(int tokens, int experts, int topk) {
    // oracle/layer_oracle.py moe_capacity: ceil(1.25 * tokens * topk / experts), to a multiple of 32
    // (a slot count the GEMM tiles need not divide; coarser rounding only adds empty rows)
    const long long c = (static_cast<long long>(tokens) * topk * 5 + 4LL * experts - 1) / (4LL * experts);
    return static_cast<int>((c + 31) / 32 * 32);
}

int moe_dense_id(int n) {
    switch (n) {
        case 0: case 1: case 2: case 4: case 5: case 6: case 7: case 8: return n;
        case 16: return 14;  // bda1 (+ loss on the last layer)
        case 20: return 20;  // bda1_bwd
        case 30: return 28;  // ln1_bwd
        case 31: return 29;  // bda0_bwd
        case 32: return 30;  // rs0_bwd_ag
        case 33: return 31;  // attn_proj_dgrad
        case 34: return 32;  // attn_proj_wgrad
        case 36: return 34;  // attn_bwd
        case 37: return 35;  // qkv_dgrad
        case 38: return 36;  // qkv_wgrad
        case 39: return 37;  // ag0_bwd_rs
        case 40: return 38;  // ln0_bwd
        default: return -1;
    }
}

namespace {

int gemm(const void* a, long long lda, bool a_mn, const void* b, long long ldb, bool b_mn, void* d,
         long long ldd, bool d_f32, int mm, int nn, int kk, bool acc, int max_ctas, cudaStream_t s,
         int epilogue = DH_EPI_NONE, void* d2 = nullptr, const void* aux0 = nullptr,
         const void* aux1 = nullptr) {
    dh_gemm_args g{};
    g.a = a;
    g.lda = lda;
    g.a_mn = a_mn;
    g.b = b;
    g.ldb = ldb;
    g.b_mn = b_mn;
    g.d = d;
    g.ldd = ldd;
    g.d_fp32 = d_f32;
    g.m = mm;
    g.n = nn;
    g.k = kk;
    g.accumulate = acc;
    g.max_ctas = max_ctas;
    g.epilogue = epilogue;
    g.d2 = d2;
    g.aux0 = aux0;
    g.aux1 = aux1;
    g.ld_aux = ldd;
    return dh_gemm(&g, s);
}

}  // namespace

int launch_moe_node(Model& m, const Op& op, cudaStream_t s, void* dy, int* dense_id) {
    *dense_id = moe_dense_id(op.node);
    if (*dense_id >= 0 || op.node >= kOptNode) {
        if (op.node >= kOptNode) *dense_id = op.node;
        return DH_OK;
    }
    const ModelCfg& k = m.cfg;
    const int H = k.hidden, T = k.tok_loc, F = k.ffn_l, E = k.experts, K = k.topk, C = k.capacity;
    const int R = k.ep * C;  // rows per local expert
    const int rows = k.moe_rows;
    const long long RH = static_cast<long long>(R) * H, RF = static_cast<long long>(R) * F;
    const long long FH = static_cast<long long>(F) * H;
    const bool a2a = k.ep > 1;
    const int cap = op.capped ? m.gemm_ctas_overlap : 0;
    Slot& sl = m.slots[op.slot];
    const LayerParams& p = m.lp[op.layer];
    auto* W = m.ptr<__nv_bfloat16>(m.w_bf16);
    auto* G = m.ptr<float>(m.w_grad);
    auto P = [&](const Buf& b) { return m.ptr<__nv_bfloat16>(b); };
    auto I = [&](const Buf& b) { return m.ptr<int>(b); };
    auto Fp = [&](const Buf& b) { return m.ptr<float>(b); };
    Comm* comm = m.ctx->comm.get();
    if ((op.node == 11 || op.node == 14 || op.node == 22 || op.node == 27) && !comm)
        return set_error(DH_ERR_CONFIG, "all-to-all node without a communicator");
    // source-side / expert-side buffers (the same buffer when there is no all-to-all)
    __nv_bfloat16* xp = a2a ? P(m.fs.xp) : P(sl.xe);
    __nv_bfloat16* ye = a2a ? P(m.fs.ye) : P(sl.y);
    __nv_bfloat16* dys = a2a ? P(m.bs.dys) : P(m.bs.dys_e);
    __nv_bfloat16* dxp = a2a ? P(m.bs.dxp) : P(m.bs.dxe);

    switch (op.node) {
        case 9:  // router
            return dh_moe_router_fwd(P(sl.ln1_full), W + p.wr, Fp(sl.probs), I(sl.ids), Fp(sl.wts), T, H, E, K, s);
        case 10:  // permute: slot assignment + gather into the source-side slot rows
            RT_TRY(dh_moe_assign(I(sl.ids), T, K, E, C, I(sl.mslot), I(sl.slot_src), s));
            return dh_moe_permute(P(sl.ln1_full), I(sl.slot_src), xp, rows, K, H, s);
        case 11:  // a2a_dispatch
            return comm->all_to_all(xp, P(sl.xe), static_cast<size_t>(C) * H, k.e_loc, false, s);
        case 12:  // expert_fc1: gate, then up with act = silu(gate) * up in its epilogue
            for (int e = 0; e < k.e_loc; ++e) {
                const __nv_bfloat16* x = P(sl.xe) + e * RH;
                __nv_bfloat16 *g = P(sl.gate) + e * RF, *u = P(sl.up) + e * RF, *a = P(sl.act) + e * RF;
                RT_TRY(gemm(x, H, false, W + p.wg + e * FH, H, false, g, F, false, R, F, H, false, cap, s));
                RT_TRY(gemm(x, H, false, W + p.wu + e * FH, H, false, u, F, false, R, F, H, false, cap, s,
                            DH_EPI_SWIGLU_FWD, a, g));
            }
            return DH_OK;
        case 13:  // expert_fc2: y = act w2^T
            for (int e = 0; e < k.e_loc; ++e)
                RT_TRY(gemm(P(sl.act) + e * RF, F, false, W + p.wd + e * FH, F, false, ye + e * RH, H, false, R,
                            H, F, false, cap, s));
            return DH_OK;
        case 14:  // a2a_combine: expert outputs back to their source ranks
            return comm->all_to_all(ye, P(sl.y), static_cast<size_t>(C) * H, k.e_loc, true, s);
        case 15:  // unpermute: weighted combine into the MLP output
            return dh_moe_unpermute(P(sl.y), I(sl.mslot), Fp(sl.wts), P(m.fs.rs_out), T, K, H, s);

        case 21:  // unpermute_bwd: per-slot gradient rows + routing-weight gradients
            return dh_moe_unpermute_bwd(dy, P(sl.y), I(sl.slot_src), Fp(sl.wts), dys, Fp(m.bs.dw), rows, K, H, s);
        case 22:  // a2a_combine_bwd (source -> expert, the dispatch layout)
            return comm->all_to_all(dys, P(m.bs.dys_e), static_cast<size_t>(C) * H, k.e_loc, false, s);
        case 23:  // expert_fc2_dgrad + SwiGLU backward in the epilogue (d_act never stored)
            for (int e = 0; e < k.e_loc; ++e)
                RT_TRY(gemm(P(m.bs.dys_e) + e * RH, H, false, W + p.wd + e * FH, F, true, P(m.bs.d_gate) + e * RF,
                            F, false, R, F, H, false, cap, s, DH_EPI_SWIGLU_BWD, P(m.bs.d_up) + e * RF,
                            P(sl.gate) + e * RF, P(sl.up) + e * RF));
            return DH_OK;
        case 24:  // expert_fc2_wgrad: dW2[e] [H,F] += dys_e^T act_e
            for (int e = 0; e < k.e_loc; ++e)
                RT_TRY(gemm(P(m.bs.dys_e) + e * RH, H, true, P(sl.act) + e * RF, F, true, G + p.wd + e * FH, F,
                            true, H, F, R, true, cap, s));
            return DH_OK;
        case 25:  // expert_fc1_dgrad: dxe = d_gate w1g + d_up w1u
            for (int e = 0; e < k.e_loc; ++e) {
                __nv_bfloat16* dx = P(m.bs.dxe) + e * RH;
                RT_TRY(gemm(P(m.bs.d_gate) + e * RF, F, false, W + p.wg + e * FH, H, true, dx, H, false, R, H, F,
                            false, cap, s));
                RT_TRY(gemm(P(m.bs.d_up) + e * RF, F, false, W + p.wu + e * FH, H, true, dx, H, false, R, H, F,
                            true, cap, s));
            }
            return DH_OK;
        case 26:  // expert_fc1_wgrad: dW1g[e], dW1u[e] [F,H] += d_{gate,up}^T xe
            for (int e = 0; e < k.e_loc; ++e) {
                const __nv_bfloat16* x = P(sl.xe) + e * RH;
                RT_TRY(gemm(P(m.bs.d_gate) + e * RF, F, true, x, H, true, G + p.wg + e * FH, H, true, F, H, R, true,
                            cap, s));
                RT_TRY(gemm(P(m.bs.d_up) + e * RF, F, true, x, H, true, G + p.wu + e * FH, H, true, F, H, R, true,
                            cap, s));
            }
            return DH_OK;
        case 27:  // a2a_dispatch_bwd (expert -> source, the combine layout)
            return comm->all_to_all(P(m.bs.dxe), dxp, static_cast<size_t>(C) * H, k.e_loc, true, s);
        case 28:  // permute_bwd: sum each token's slot gradients (into ln1_bwd's input)
            return dh_moe_permute_bwd(dxp, I(sl.mslot), P(m.bs.rs_out), T, K, H, s);
        case 29:  // router_bwd: adds the routing path (tensor-core GEMMs) to dL/d ln1 in place
            return dh_moe_router_bwd(Fp(sl.probs), I(sl.ids), I(sl.mslot), Fp(m.bs.dw), P(sl.ln1_full), W + p.wr,
                                     P(m.bs.rs_out), P(m.bs.rs_out), G + p.wr, Fp(m.bs.router_scratch), T, H, E,
                                     K, s);
        default:
            return set_error(DH_ERR_CONFIG, "launch_moe_node: unknown moe_ep node " + std::to_string(op.node));
    }
}

}  // namespace dh
