// Llama TP+SP layer stack on one rank: pool layout, parameter init and the
// per-template-node launchers.
//
// Node ids / names are the dense_tp_sp template (reference op_model.cpp:79-113):
//   fwd  0 ln0  1 ag0  2 qkv(+RoPE)  4 attn  5 attn_proj  6 rs0  7 bda0  8 ln1
//        9 ag1  10 mlp_gate  11 mlp_up  12 mlp_down(SwiGLU + GEMM)  13 rs1  14 bda1
//   bwd 20 bda1_bwd  21 rs1_bwd_ag  22 mlp_down_dgrad(+SwiGLU bwd)  23 mlp_down_wgrad
//       24 mlp_gate_dgrad  25 mlp_up_dgrad  26 mlp_fc1_wgrad  27 ag1_bwd_rs  28 ln1_bwd
//       29 bda0_bwd  30 rs0_bwd_ag  31 attn_proj_dgrad  32 attn_proj_wgrad
//       34 attn_bwd(+RoPE bwd)  35 qkv_dgrad  36 qkv_wgrad  37 ag0_bwd_rs  38 ln0_bwd
//
// Megatron TP+SP partitioning: W_qkv, W_gate, W_up column-parallel (local q
// heads n_heads/tp, kv heads n_kv/tp, ffn/tp rows); W_o, W_down row-parallel;
// RMSNorm and the residual run on the [seq/tp, hidden] sequence shard. The
// gathered LN outputs are saved for the wgrad GEMMs (SURVEY §8(a) build note i).
// With tp == 1 the collective nodes do not exist and producers write straight
// into their consumers' buffers.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "runtime.hpp"

namespace dh {

namespace {

struct Pool {
    size_t cursor = 0;
    std::map<std::string, size_t>* usage;
    Buf take(size_t bytes, const char* cat) {
        Buf b;
        b.off = cursor;
        b.bytes = bytes;
        cursor += (bytes + 255) & ~static_cast<size_t>(255);
        (*usage)[cat] += bytes;
        return b;
    }
};

unsigned long long mix(unsigned long long a, unsigned long long b) {
    unsigned long long z = a * 0x9E3779B97F4A7C15ull + b + 0x632BE59BD9B4E019ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace

int derive_cfg(const dh_model_cfg* c, int tp, int rank, ModelCfg* out) {
    ModelCfg k;
    k.hidden = c->hidden;
    k.ffn = c->ffn;
    k.n_heads = c->n_heads;
    k.n_kv_heads = c->n_kv_heads;
    k.head_dim = c->head_dim;
    k.layers = c->layers;
    k.seq = c->seq_len;
    k.micro_batches = c->micro_batches;
    k.rope_theta = c->rope_theta;
    k.eps = c->norm_eps;
    k.seed = c->seed;
    k.init_std = c->init_std;
    k.slots = c->slots;
    k.split = c->split_layer;
    k.pp_rank = c->pp_rank;
    k.pp_size = c->pp_size > 0 ? c->pp_size : 1;
    k.tp = tp;
    k.rank = rank;
    if (c->experts > 1) {
        // MoE: the group is the EP group; attention and the router run
        // data-parallel (TP = 1) on this rank's own micro-batches
        k.moe = true;
        k.experts = c->experts;
        k.topk = c->topk > 0 ? c->topk : 2;
        k.ep = tp;
        k.ep_rank = rank;
        k.tp = 1;
        k.rank = 0;
        if (k.topk > k.experts || k.topk > 8 || k.experts > 64)
            return set_error(DH_ERR_CONFIG, "model: MoE needs topk <= min(8, experts), experts <= 64");
        if (k.experts % k.ep) return set_error(DH_ERR_INFEASIBLE, "model: experts must be divisible by the EP size");
        k.e_loc = k.experts / k.ep;
        k.capacity = c->capacity > 0 ? c->capacity : moe_capacity(c->seq_len, k.experts, k.topk);
        k.moe_rows = k.experts * k.capacity;
    }
    k.seq_full = c->seq_len;
    if (c->context_parallel) {
        if (c->experts > 1) return set_error(DH_ERR_CONFIG, "model: context parallelism is dense-only");
        k.cp = tp;
        k.cp_rank = rank;
        k.tp = 1;
        k.rank = 0;
        if (c->seq_len % (256 * k.cp))
            return set_error(DH_ERR_INFEASIBLE, "model: context parallelism needs seq_len % (256 * group size) == 0");
        k.seq = c->seq_len / k.cp;
    }
    if (k.split < 0 || k.split >= c->layers || k.slots < 0 || k.pp_rank < 0 || k.pp_rank >= k.pp_size)
        return set_error(DH_ERR_CONFIG, "model: bad pipeline stage fields (split_layer, slots, pp_rank/pp_size)");
    if (k.hidden <= 0 || k.layers <= 0 || k.seq <= 0 || k.micro_batches < 1 || k.head_dim <= 0 ||
        k.n_heads <= 0 || k.n_kv_heads <= 0 || tp < 1)
        return set_error(DH_ERR_CONFIG, "model: dimensions must be positive");
    if (k.seq % k.tp || k.n_heads % k.tp || k.n_kv_heads % k.tp || k.ffn % k.tp)
        return set_error(DH_ERR_INFEASIBLE,
                         "model: seq, n_heads, n_kv_heads and ffn must be divisible by tp");
    if (k.n_heads % k.n_kv_heads) return set_error(DH_ERR_CONFIG, "model: n_heads % n_kv_heads");
    if (k.head_dim != 64 && k.head_dim != 128)
        return set_error(DH_ERR_CONFIG, "model: head_dim must be 64 or 128");
    if (k.hidden % 256 || (k.ffn / k.tp) % 64)
        return set_error(DH_ERR_CONFIG, "model: hidden % 256 and (ffn/tp) % 64 required");
    k.tok_loc = k.seq / k.tp;
    k.nq_l = k.n_heads / k.tp;
    k.nkv_l = k.n_kv_heads / k.tp;
    k.qkv_n = (k.nq_l + 2 * k.nkv_l) * k.head_dim;
    k.attn_n = k.nq_l * k.head_dim;
    k.ffn_l = k.ffn / k.tp;
    *out = k;
    return DH_OK;
}

weft::ClusterSpec default_cluster() {
    weft::ClusterSpec cl;
    cl.name = "b200";
    cl.gpus = 8;
    cl.per_node = 8;
    cl.peak_tflops = 2250.0;
    cl.local_bw_gbs = 900.0;
    cl.cross_bw_gbs = 50.0;
    cl.mem_gb = 180.0;
    return cl;
}

// The layer DAG from the same template and specs the planner uses.
int build_dags(Model& m, const weft::ClusterSpec& cl, const weft::SoloTimeTable* solo) {
    weft::ModelSpec ms;
    ms.name = "dh-llama";
    ms.family = weft::ModelFamily::llama;
    ms.hidden = m.cfg.hidden;
    ms.intermediate = m.cfg.ffn;
    ms.layers = m.cfg.layers;
    ms.seq_len = m.cfg.seq_full;  // the template's node costs use seq / cp per rank
    weft::ParallelismSpec par;
    par.tp = m.cfg.tp;
    par.sp = m.cfg.tp > 1;
    par.cp = m.cfg.cp;  // cp > 1 activates cp_kv_exchange / cp_kv_exchange_bwd
    if (m.cfg.moe) {  // moe_ep template (reference op_model.cpp:410)
        ms.name = "dh-moe";
        ms.family = weft::ModelFamily::phi_moe;
        ms.experts = m.cfg.experts;
        ms.topk = m.cfg.topk;
        par.ep = m.cfg.ep;
        par.dp = m.cfg.ep;  // the EP group is a subset of the DP group (presets.cpp validate)
    }
    try {
        auto dags = weft::build_layer_dag(ms, par, cl, solo);
        m.fwd_dag = std::move(dags.first);
        m.bwd_dag = std::move(dags.second);
    } catch (const std::exception& e) {
        return set_error(DH_ERR_CONFIG, e.what());
    }
    return DH_OK;
}

int model_create(Ctx* ctx, const dh_model_cfg* c, Model** out) {
    auto m = std::make_unique<Model>();
    m->ctx = ctx;
    RT_TRY(derive_cfg(c, ctx->tp_size, ctx->tp_rank, &m->cfg));
    ModelCfg& k = m->cfg;

    const size_t H = k.hidden, S = k.seq, T = k.tok_loc, Q = k.qkv_n, A = k.attn_n, F = k.ffn_l;
    const int L = k.layers;

    // ---- parameters: gammas first (contiguous, for the SP all-reduce), then
    // per-layer matrices, each 128-element aligned.
    auto al = [](size_t n) { return (n + 127) & ~static_cast<size_t>(127); };
    size_t off = 0;
    m->lp.resize(L);
    for (int l = 0; l < L; ++l) {
        m->lp[l].g0 = off;
        off += al(H);
        m->lp[l].g1 = off;
        off += al(H);
    }
    m->gamma_elems = off;
    for (int l = 0; l < L; ++l) {
        m->lp[l].wqkv = off;
        off += al(Q * H);
        m->lp[l].wo = off;
        off += al(H * A);
        const size_t ex = k.moe ? static_cast<size_t>(k.e_loc) : 1;  // stacked local experts
        m->lp[l].wr = off;
        off += k.moe ? al(static_cast<size_t>(k.experts) * H) : 0;
        m->lp[l].wg = off;
        off += al(ex * F * H);
        m->lp[l].wu = off;
        off += al(ex * F * H);
        m->lp[l].wd = off;
        off += al(ex * H * F);
    }
    m->n_params = off;

    Pool pool{0, &m->usage};
    m->w_bf16 = pool.take(off * 2, "state.weights_bf16");
    m->w_master = pool.take(off * 4, "state.master_fp32");
    m->w_grad = pool.take(off * 4, "state.grad_fp32");
    m->adam_m = pool.take(off * 4, "state.adam_m");
    m->adam_v = pool.take(off * 4, "state.adam_v");

    // MLP rows: tokens (dense) or this rank's expert slot rows (MoE)
    const size_t MR = k.moe ? static_cast<size_t>(k.moe_rows) : S;
    const size_t E = k.experts, K = k.topk;
    m->slots.resize(k.slots > 0 ? k.slots : L + 1);
    for (auto& s : m->slots) {
        s.out = pool.take(T * H * 2, "act.slots");
        s.rstd0 = pool.take(T * 4, "act.slots");
        s.ln0_full = pool.take(S * H * 2, "act.slots");
        s.qkv = pool.take(S * Q * 2, "act.slots");
        s.o = pool.take(S * A * 2, "act.slots");
        s.lse = pool.take(S * k.nq_l * 4, "act.slots");
        s.x1 = pool.take(T * H * 2, "act.slots");
        s.rstd1 = pool.take(T * 4, "act.slots");
        s.ln1_full = pool.take(S * H * 2, "act.slots");
        s.gate = pool.take(MR * F * 2, "act.slots");
        s.up = pool.take(MR * F * 2, "act.slots");
        s.act = pool.take(MR * F * 2, "act.slots");
        if (k.moe) {
            s.probs = pool.take(T * E * 4, "act.slots");
            s.ids = pool.take(T * K * 4, "act.slots");
            s.wts = pool.take(T * K * 4, "act.slots");
            s.mslot = pool.take(T * K * 4, "act.slots");
            s.slot_src = pool.take(MR * 4, "act.slots");
            s.xe = pool.take(MR * H * 2, "act.slots");
            s.y = pool.take(MR * H * 2, "act.slots");
        }
    }
    const bool tp1 = k.tp == 1;
    m->fs.ln_loc = pool.take(tp1 ? 0 : T * H * 2, "act.fwd_transient");
    m->fs.part = pool.take(tp1 ? 0 : S * H * 2, "act.fwd_transient");
    m->fs.rs_out = pool.take(T * H * 2, "act.fwd_transient");
    const bool a2a = k.moe && k.ep > 1;
    const size_t KV = 2 * static_cast<size_t>(k.nkv_l) * k.head_dim;  // K|V columns
    const size_t SF = k.cp > 1 ? static_cast<size_t>(k.seq_full) : 0;
    m->fs.kv_loc = pool.take(SF ? S * KV * 2 : 0, "act.fwd_transient");
    m->fs.kv_full = pool.take(SF * KV * 2, "act.fwd_transient");
    m->fs.xp = pool.take(a2a ? MR * H * 2 : 0, "act.fwd_transient");
    m->fs.ye = pool.take(a2a ? MR * H * 2 : 0, "act.fwd_transient");
    auto& b = m->bs;
    b.grad[0] = pool.take(T * H * 2, "act.bwd_transient");
    b.grad[1] = pool.take(T * H * 2, "act.bwd_transient");
    b.d_x1 = pool.take(T * H * 2, "act.bwd_transient");
    for (int i = 0; i < 2; ++i) b.dy_full[i] = pool.take(tp1 ? 0 : S * H * 2, "act.bwd_transient");
    b.d_gate = pool.take(MR * F * 2, "act.bwd_transient");
    b.d_up = pool.take(MR * F * 2, "act.bwd_transient");
    if (k.moe) {
        b.dys = pool.take(a2a ? MR * H * 2 : 0, "act.bwd_transient");
        b.dys_e = pool.take(MR * H * 2, "act.bwd_transient");
        b.dxe = pool.take(MR * H * 2, "act.bwd_transient");
        b.dxp = pool.take(a2a ? MR * H * 2 : 0, "act.bwd_transient");
        b.dw = pool.take(T * K * 4, "act.bwd_transient");
        b.router_scratch = pool.take(
            static_cast<size_t>(dh_moe_router_bwd_scratch_floats(static_cast<int>(T), static_cast<int>(H),
                                                                 static_cast<int>(E))) * 4,
            "act.bwd_transient");
    }
    {
        // SwiGLU runs in the mlp GEMM epilogues by default. Measured on B200 the
        // standalone kernels after plain GEMMs were no faster even at TP=8
        // (1.5 waves of 256x256 pair tiles, where the epilogue is least hidden)
        // and lost overlap under SI; DH_SWIGLU_EPILOGUE=0 selects them.
        const char* env = std::getenv("DH_SWIGLU_EPILOGUE");
        m->swiglu_in_epilogue = env ? std::atoi(env) != 0 : true;
        // mlp_gate | mlp_up as one GEMM and the two dgrads as one only without
        // tensor parallelism: at TP = 8 (emulated collectives, 32 layers x 8
        // micro-batches) merging cut the compute-only step 214 -> 209 ms but the
        // SI step rose 230.4 -> 235.1 ms (hidden comm 0.81 -> 0.69): the coarser
        // GEMMs leave the plan fewer places to start the other strand's
        // collectives. DH_MLP_MERGE=0/1 overrides.
        const char* mm = std::getenv("DH_MLP_MERGE");
        m->mlp_merge = mm ? std::atoi(mm) != 0 : k.tp == 1;
        if (!m->swiglu_in_epilogue) b.d_act = pool.take(MR * F * 2, "act.bwd_transient");
    }
    b.dx_part = pool.take(tp1 ? 0 : S * H * 2, "act.bwd_transient");
    b.dx1_full = pool.take(tp1 ? 0 : S * H * 2, "act.bwd_transient");
    b.d_o = pool.take(S * A * 2, "act.bwd_transient");
    b.dqkv = pool.take(S * Q * 2, "act.bwd_transient");
    b.kv_loc = pool.take(SF ? S * KV * 2 : 0, "act.bwd_transient");
    b.kv_full = pool.take(SF * KV * 2, "act.bwd_transient");
    b.dkv_full = pool.take(SF * KV * 2, "act.bwd_transient");
    b.dkv_loc = pool.take(SF ? S * KV * 2 : 0, "act.bwd_transient");
    {
        const int SK = SF ? k.seq_full : static_cast<int>(S), qoff = k.cp_rank * static_cast<int>(S);
        const size_t bwd = static_cast<size_t>(
            dh_attn_bwd_scratch_floats_ex(static_cast<int>(S), k.nq_l, k.nkv_l, k.head_dim, SK, SF ? qoff : 0));
        const size_t fwd = static_cast<size_t>(
            dh_attn_fwd_scratch_floats_ex(static_cast<int>(S), k.nq_l, k.nkv_l, k.head_dim, SK, SF ? qoff : 0));
        b.attn_scratch = pool.take(std::max(bwd, fwd) * 4, "act.bwd_transient");
    }
    b.ln_partial = pool.take(std::min<size_t>(T, 1184) * H * 4, "act.bwd_transient");
    b.rs_out = pool.take(T * H * 2, "act.bwd_transient");
    for (int i = 0; i < k.micro_batches; ++i) {
        m->mb_in.push_back(pool.take(T * H * 2, "io.inputs"));
        m->mb_dy.push_back(pool.take(T * H * 2, "io.inputs"));
        if (k.split > 0) {
            m->mid_in.push_back(pool.take(T * H * 2, "io.stage"));
            m->mid_dy.push_back(pool.take(T * H * 2, "io.stage"));
        }
    }
    m->loss = pool.take(std::max(k.micro_batches, 1) * 4 + 1024 * 4, "io.loss");
    m->opt_hp = pool.take(64, "io.optim");

    m->pool_bytes = pool.cursor;
    RT_CUDA(cudaSetDevice(ctx->device));
    RT_CUDA(cudaMalloc(&m->base, m->pool_bytes));
    RT_CUDA(cudaMemset(m->base, 0, m->pool_bytes));

    // ---- deterministic synthetic init (tests overwrite through dh_model_tensor)
    cudaStream_t s = ctx->lane[0];
    auto* wb = m->ptr<__nv_bfloat16>(m->w_bf16);
    auto* wm = m->ptr<float>(m->w_master);
    std::vector<float> ones(H, 1.f);
    for (int l = 0; l < L; ++l) {
        const LayerParams& p = m->lp[l];
        RT_TRY(dh_fill_bf16(wb + p.g0, 1.f, H, s));
        RT_TRY(dh_fill_bf16(wb + p.g1, 1.f, H, s));
        RT_CUDA(cudaMemcpyAsync(wm + p.g0, ones.data(), H * 4, cudaMemcpyHostToDevice, s));
        RT_CUDA(cudaMemcpyAsync(wm + p.g1, ones.data(), H * 4, cudaMemcpyHostToDevice, s));
        if (k.moe) {
            // replicated (data-parallel) attention / router weights: the same on
            // every EP rank; expert matrices seeded by their global expert id
            const std::pair<size_t, size_t> rep[] = {{p.wqkv, Q * H}, {p.wo, H * A}, {p.wr, E * H}};
            for (int t = 0; t < 3; ++t)
                RT_TRY(dh_init_normal(wb + rep[t].first, wm + rep[t].first, rep[t].second,
                                      mix(k.seed, l * 16 + t), k.init_std, s));
            for (int e = 0; e < k.e_loc; ++e) {
                const int ge = k.ep_rank * k.e_loc + e;
                const std::pair<size_t, size_t> mats[] = {
                    {p.wg + e * F * H, F * H}, {p.wu + e * F * H, F * H}, {p.wd + e * H * F, H * F}};
                for (int t = 0; t < 3; ++t)
                    RT_TRY(dh_init_normal(wb + mats[t].first, wm + mats[t].first, mats[t].second,
                                          mix(mix(k.seed, l * 16 + 8 + t), 4096 + ge), k.init_std, s));
            }
            continue;
        }
        const std::pair<size_t, size_t> mats[] = {
            {p.wqkv, Q * H}, {p.wo, H * A}, {p.wg, F * H}, {p.wu, F * H}, {p.wd, H * F}};
        for (int t = 0; t < 5; ++t) {
            const unsigned long long sd = mix(mix(k.seed, l * 16 + t), k.rank);
            RT_TRY(dh_init_normal(wb + mats[t].first, wm + mats[t].first, mats[t].second, sd,
                                  k.init_std, s));
        }
    }
    for (int i = 0; i < k.micro_batches; ++i) {
        const int r = k.moe ? k.ep_rank : k.rank;  // MoE ranks see different data
        RT_TRY(dh_init_normal(m->ptr(m->mb_in[i]), nullptr, T * H, mix(mix(k.seed, 1000 + i), r), 1.f, s));
        RT_TRY(dh_init_normal(m->ptr(m->mb_dy[i]), nullptr, T * H, mix(mix(k.seed, 2000 + i), r), 1.f, s));
    }
    RT_CUDA(cudaStreamSynchronize(s));

    RT_TRY(build_dags(*m, default_cluster(), nullptr));
    // EP > 1: replicated weights need their data-parallel gradient all-reduce
    // before AdamW, so the optimizer runs after the program
    if ((k.moe && k.ep > 1) || k.cp > 1) m->fuse_optimizer = false;
    *out = m.release();
    return DH_OK;
}

void model_destroy(Model* m) {
    if (!m) return;
    cudaSetDevice(m->ctx->device);
    if (m->graph) cudaGraphExecDestroy(m->graph);
    for (auto e : m->events)
        if (e) cudaEventDestroy(e);
    for (auto e : m->fork_join)
        if (e) cudaEventDestroy(e);
    if (m->base) cudaFree(m->base);
    delete m;
}

// ------------------------------------------------------------------ node launchers

namespace {

dh_gemm_args gemm_args(const void* a, long long lda, bool a_mn, const void* b, long long ldb, bool b_mn, void* d,
                       long long ldd, bool d_f32, int mm, int nn, int kk, bool acc, int max_ctas) {
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
    g.ld_aux = ldd;
    return g;
}

int gemm(const void* a, long long lda, bool a_mn, const void* b, long long ldb, bool b_mn, void* d,
         long long ldd, bool d_f32, int mm, int nn, int kk, bool acc, int max_ctas,
         cudaStream_t s, int epilogue = DH_EPI_NONE, void* d2 = nullptr, const void* aux0 = nullptr,
         const void* aux1 = nullptr) {
    dh_gemm_args g{};
    g.epilogue = epilogue;
    g.d2 = d2;
    g.aux0 = aux0;
    g.aux1 = aux1;
    g.ld_aux = ldd;
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
    return dh_gemm(&g, s);
}

}  // namespace

// Transfer tag: activations and gradients of a micro-batch travel on separate
// channels (a stage may send one before it receives the other).
int xfer_tag(const Op& op) {
    const bool act = op.node == kSendAct || op.node == kRecvAct;
    return (act ? 0 : 1) + 2 * op.strand;
}

// Context parallelism: pack this chunk's post-RoPE K|V columns (a strided view
// of the slot's qkv rows) and all-gather them over the CP group; rank r's rows
// land at [r * seq, (r + 1) * seq), i.e. in global position order.
int cp_gather_kv(Model& m, const Slot& sl, const Buf& kv_loc, const Buf& kv_full, cudaStream_t s) {
    const ModelCfg& k = m.cfg;
    const size_t D = k.head_dim, Q = k.qkv_n, KV = 2 * static_cast<size_t>(k.nkv_l) * D;
    RT_CUDA(cudaMemcpy2DAsync(m.ptr(kv_loc), KV * 2, m.ptr<__nv_bfloat16>(sl.qkv) + k.nq_l * D, Q * 2, KV * 2,
                              static_cast<size_t>(k.seq), cudaMemcpyDeviceToDevice, s));
    return m.ctx->comm->all_gather(m.ptr(kv_loc), m.ptr(kv_full), static_cast<size_t>(k.seq) * KV, s);
}

int launch_node(Model& m, const Op& op, cudaStream_t s) {
    const ModelCfg& k = m.cfg;
    const int H = k.hidden, S = k.seq, T = k.tok_loc, Q = k.qkv_n, A = k.attn_n, F = k.ffn_l;
    const int D = k.head_dim;
    const long long TH = static_cast<long long>(T) * H;
    const bool tp1 = k.tp == 1;
    const int cap = op.capped ? m.gemm_ctas_overlap : 0;
    Slot& sl = m.slots[op.slot < 0 ? 0 : op.slot];  // (optimizer ops own no slot)
    const LayerParams& p = m.lp[op.layer];
    auto* W = m.ptr<__nv_bfloat16>(m.w_bf16);
    auto* G = m.ptr<float>(m.w_grad);
    auto P = [&](const Buf& b) { return m.ptr(b); };
    // a split stage's way-back half starts from the activation the next stage sent
    // (strand -1: the per-layer optimizer op, which reads no activations)
    const bool act = op.strand >= 0;
    void* x_in = !act                                   ? nullptr
                 : k.split > 0 && op.layer == k.split   ? P(m.mid_in[op.strand])
                 : op.prev_slot < 0                     ? P(m.mb_in[op.strand])
                                                        : P(m.slots[op.prev_slot].out);
    const float scale = 1.f / std::sqrt(static_cast<float>(D));
    // backward running-gradient ping-pong (see header of executor.cpp)
    const int L = k.layers;
    void* dy = !act                                      ? nullptr
               : op.layer == L - 1                         ? P(m.mb_dy[op.strand])
               : k.split > 0 && op.layer == k.split - 1    ? P(m.mid_dy[op.strand])
                                                           : P(m.bs.grad[(L - 2 - op.layer) & 1]);
    void* d_x = P(m.bs.grad[(L - 1 - op.layer) & 1]);
    Comm* comm = m.ctx->comm.get();
    auto need_comm = [&]() -> int {
        return comm ? DH_OK : set_error(DH_ERR_CONFIG, "collective node without a communicator");
    };

    int node = op.node;
    if (k.moe) {
        int dense = -1;
        RT_TRY(launch_moe_node(m, op, s, dy, &dense));
        if (dense < 0) return DH_OK;  // an MoE node, launched
        node = dense;
    }
    switch (node) {
        // ---------------------------------------------------------------- forward
        case 0:  // ln0
            return dh_rmsnorm_fwd(x_in, W + p.g0, tp1 ? P(sl.ln0_full) : P(m.fs.ln_loc),
                                  m.ptr<float>(sl.rstd0), T, H, k.eps, s);
        case 1:  // ag0
            RT_TRY(need_comm());
            return comm->all_gather(P(m.fs.ln_loc), P(sl.ln0_full), TH, s);
        case 2:  // qkv (+ RoPE on q, k at the chunk's global positions)
            RT_TRY(gemm(P(sl.ln0_full), H, false, W + p.wqkv, H, false, P(sl.qkv), Q, false, S, Q, H,
                        false, cap, s));
            return dh_rope(P(sl.qkv), Q, S, k.nq_l, k.nkv_l, D, k.rope_theta, k.cp_rank * S, 0, s);
        case 3:  // cp_kv_exchange: all-gather the group's K|V rows (position order)
            RT_TRY(need_comm());
            return cp_gather_kv(m, sl, m.fs.kv_loc, m.fs.kv_full, s);
        case 4: {  // attn
            auto* qkv = m.ptr<__nv_bfloat16>(sl.qkv);
            if (k.cp > 1) {  // this chunk's queries against every key up to them
                auto* kv = m.ptr<__nv_bfloat16>(m.fs.kv_full);
                return dh_attn_fwd_ex(qkv, kv, kv + k.nkv_l * D, Q, 2LL * k.nkv_l * D, P(sl.o), A,
                                      m.ptr<float>(sl.lse), m.ptr<float>(m.bs.attn_scratch),
                                      static_cast<long long>(m.bs.attn_scratch.bytes / 4), S, k.seq_full,
                                      k.cp_rank * S, k.nq_l, k.nkv_l, D, scale, s);
            }
            // the transient attention scratch is shared with attn_bwd: both run on the compute lane
            return dh_attn_fwd(qkv, qkv + k.nq_l * D, qkv + (k.nq_l + k.nkv_l) * D, Q, Q, P(sl.o), A,
                               m.ptr<float>(sl.lse), m.ptr<float>(m.bs.attn_scratch),
                               static_cast<long long>(m.bs.attn_scratch.bytes / 4), S, k.nq_l, k.nkv_l,
                               D, scale, s);
        }
        case 5:  // attn_proj (row-parallel: partial sums before the reduce-scatter)
            return gemm(P(sl.o), A, false, W + p.wo, A, false, tp1 ? P(m.fs.rs_out) : P(m.fs.part), H,
                        false, S, H, A, false, cap, s);
        case 6:  // rs0
            RT_TRY(need_comm());
            return comm->reduce_scatter(P(m.fs.part), P(m.fs.rs_out), TH, s);
        case 7:  // bda0: x1 = x + attn_out, fused with ln1 (its only consumer, next in
            // every forward order): one pass writes x1 and ln1's output
            return dh_add_rmsnorm_fwd(x_in, P(m.fs.rs_out), P(sl.x1), W + p.g1,
                                      tp1 ? P(sl.ln1_full) : P(m.fs.ln_loc), m.ptr<float>(sl.rstd1), T, H, k.eps, s);
        case 8:  // ln1: computed by bda0's fused kernel
            return DH_OK;
        case 9:  // ag1
            RT_TRY(need_comm());
            return comm->all_gather(P(m.fs.ln_loc), P(sl.ln1_full), TH, s);
        case 10:    // mlp_gate
        case 11: {  // mlp_up
            if (m.swiglu_in_epilogue && m.mlp_merge) {
                // the earlier of the two computes gate, up and act = silu(gate) * up in one
                // GEMM (the CTA pair's B halves are Wg and Wu rows of the same features);
                // the later launches nothing
                if (op.fuse_swiglu) return DH_OK;
                dh_gemm_args g = gemm_args(P(sl.ln1_full), H, false, W + p.wg, H, false, P(sl.gate), F, false, S, F,
                                           H, false, cap);
                g.epilogue = DH_EPI_SWIGLU_PAIR;
                g.b2 = W + p.wu;
                g.ldb2 = H;
                g.d2 = P(sl.up);
                g.d_m2 = P(sl.act);
                return dh_gemm(&g, s);
            }
            const bool gate = op.node == 10;
            // unmerged: the later of the two applies SwiGLU in its epilogue
            const bool epi = op.fuse_swiglu && m.swiglu_in_epilogue;
            RT_TRY(gemm(P(sl.ln1_full), H, false, W + (gate ? p.wg : p.wu), H, false, P(gate ? sl.gate : sl.up), F,
                        false, S, F, H, false, cap, s,
                        epi ? (gate ? DH_EPI_SWIGLU_FWD_UP : DH_EPI_SWIGLU_FWD) : DH_EPI_NONE, P(sl.act),
                        P(gate ? sl.up : sl.gate)));
            if (op.fuse_swiglu && !epi)
                return dh_swiglu_fwd(P(sl.gate), P(sl.up), P(sl.act), static_cast<long long>(S) * F, s);
            return DH_OK;
        }
        case 12:  // mlp_down (row-parallel; act was produced by the mlp_gate/mlp_up epilogue)
            return gemm(P(sl.act), F, false, W + p.wd, F, false, tp1 ? P(m.fs.rs_out) : P(m.fs.part),
                        H, false, S, H, F, false, cap, s);
        case 13:  // rs1
            RT_TRY(need_comm());
            return comm->reduce_scatter(P(m.fs.part), P(m.fs.rs_out), TH, s);
        case 14:  // bda1: out = x1 + mlp_out (+ loss on the last layer)
            RT_TRY(dh_add(P(sl.x1), P(m.fs.rs_out), P(sl.out), TH, s));
            if (op.layer == L - 1) {
                float* loss = m.ptr<float>(m.loss);
                return dh_dot_loss(P(sl.out), P(m.mb_dy[op.strand]), TH, loss + k.micro_batches,
                                   loss + op.strand, s);
            }
            return DH_OK;

        // ---------------------------------------------------------------- backward
        case 20:  // bda1_bwd: residual gradient pass-through. No kernel: ln1_bwd joins
            // the skip gradient straight from dy (still intact then: the running-gradient
            // ping-pong rewrites dy only at the next layer's ln0_bwd)
            return DH_OK;
        case 21:  // rs1_bwd_ag
            RT_TRY(need_comm());
            return comm->all_gather(dy, P(m.bs.dy_full[op.layer & 1]), TH, s);
        case 22: {  // mlp_down_dgrad + SwiGLU backward (in its epilogue: d_act never stored)
            const void* dyf = tp1 ? dy : P(m.bs.dy_full[op.layer & 1]);
            if (m.swiglu_in_epilogue)
                return gemm(dyf, H, false, W + p.wd, F, true, P(m.bs.d_gate), F, false, S, F, H, false, cap, s,
                            DH_EPI_SWIGLU_BWD, P(m.bs.d_up), P(sl.gate), P(sl.up));
            RT_TRY(gemm(dyf, H, false, W + p.wd, F, true, P(m.bs.d_act), F, false, S, F, H, false, cap, s));
            return dh_swiglu_bwd(P(sl.gate), P(sl.up), P(m.bs.d_act), P(m.bs.d_gate), P(m.bs.d_up),
                                 static_cast<long long>(S) * F, s);
        }
        case 23: {  // mlp_down_wgrad: dWd[H,F] += dY^T act
            const void* dyf = tp1 ? dy : P(m.bs.dy_full[op.layer & 1]);
            return gemm(dyf, H, true, P(sl.act), F, true, G + p.wd, F, true, H, F, S, true, cap, s);
        }
        case 24:    // mlp_gate_dgrad
        case 25: {  // mlp_up_dgrad: whichever runs first computes both, dX = d_gate Wg + d_up Wu,
            // as one K-concatenated GEMM (one pass, one rounding); the other launches nothing
            if (!m.mlp_merge)
                return gemm(op.node == 24 ? P(m.bs.d_gate) : P(m.bs.d_up), F, false, W + (op.node == 24 ? p.wg : p.wu),
                            H, true, tp1 ? P(m.bs.rs_out) : P(m.bs.dx_part), H, false, S, H, F, !op.first_dx, cap, s);
            if (!op.first_dx) return DH_OK;
            dh_gemm_args g = gemm_args(P(m.bs.d_gate), F, false, W + p.wg, H, true,
                                       tp1 ? P(m.bs.rs_out) : P(m.bs.dx_part), H, false, S, H, F, false, cap);
            g.a2 = P(m.bs.d_up);
            g.lda2 = F;
            g.b2 = W + p.wu;
            g.ldb2 = H;
            g.k2 = F;
            return dh_gemm(&g, s);
        }
        case 26: {  // mlp_fc1_wgrad: dWg, dWu [F,H] += d_{gate,up}^T ln1, one M-concatenated GEMM
            if (op.part >= 0) {  // one of the two (the executor placed them under different collectives)
                dh_gemm_args g = gemm_args(P(op.part ? m.bs.d_up : m.bs.d_gate), F, true, P(sl.ln1_full), H, true,
                                           G + (op.part ? p.wu : p.wg), H, true, F, H, S, true, cap);
                return dh_gemm(&g, s);
            }
            dh_gemm_args g = gemm_args(P(m.bs.d_gate), F, true, P(sl.ln1_full), H, true, G + p.wg, H, true, F, H, S,
                                       true, cap);
            g.a2 = P(m.bs.d_up);
            g.lda2 = F;
            g.m2 = F;
            g.d_m2 = G + p.wu;
            g.ldd_m2 = H;
            return dh_gemm(&g, s);
        }
        case 27:  // ag1_bwd_rs
            RT_TRY(need_comm());
            return comm->reduce_scatter(P(m.bs.dx_part), P(m.bs.rs_out), TH, s);
        case 28:  // ln1_bwd (+ residual join: d_x1 = RMSNorm'(.) + dy)
            return dh_rmsnorm_bwd(P(sl.x1), W + p.g1, m.ptr<float>(sl.rstd1), P(m.bs.rs_out),
                                  dy, P(m.bs.d_x1), G + p.g1, m.ptr<float>(m.bs.ln_partial),
                                  T, H, s);
        case 29:  // bda0_bwd: skip-connection gradient to the layer input. No kernel:
            // ln0_bwd joins it from d_x1 (rewritten only by the next layer's ln1_bwd)
            return DH_OK;
        case 30:  // rs0_bwd_ag
            RT_TRY(need_comm());
            return comm->all_gather(P(m.bs.d_x1), P(m.bs.dx1_full), TH, s);
        case 31: {  // attn_proj_dgrad: d_o = dX1 Wo
            const void* src = tp1 ? P(m.bs.d_x1) : P(m.bs.dx1_full);
            return gemm(src, H, false, W + p.wo, A, true, P(m.bs.d_o), A, false, S, A, H, false, cap, s);
        }
        case 32: {  // attn_proj_wgrad: dWo[H,A] += dX1^T o
            const void* src = tp1 ? P(m.bs.d_x1) : P(m.bs.dx1_full);
            return gemm(src, H, true, P(sl.o), A, true, G + p.wo, A, true, H, A, S, true, cap, s);
        }
        case 33:  // cp_kv_exchange_bwd: re-gather K|V for attn_bwd (the slot keeps only this chunk's)
            RT_TRY(need_comm());
            return cp_gather_kv(m, sl, m.bs.kv_loc, m.bs.kv_full, s);
        case 34: {  // attn_bwd (+ RoPE bwd on dq, dk)
            auto* qkv = m.ptr<__nv_bfloat16>(sl.qkv);
            auto* dqkv = m.ptr<__nv_bfloat16>(m.bs.dqkv);
            if (k.cp > 1) {
                // dK|dV over every key from this chunk's queries, then reduce-scattered
                // to the owners (rank-order sum) and unpacked into dqkv's K|V columns
                RT_TRY(need_comm());
                auto* kv = m.ptr<__nv_bfloat16>(m.bs.kv_full);
                auto* dkv = m.ptr<__nv_bfloat16>(m.bs.dkv_full);
                const long long KV = 2LL * k.nkv_l * D;
                RT_TRY(dh_attn_bwd_ex(qkv, kv, kv + k.nkv_l * D, Q, KV, P(sl.o), A, m.ptr<float>(sl.lse),
                                      P(m.bs.d_o), dqkv, dkv, dkv + k.nkv_l * D, Q, KV,
                                      m.ptr<float>(m.bs.attn_scratch), S, k.seq_full, k.cp_rank * S, k.nq_l,
                                      k.nkv_l, D, scale, s));
                RT_TRY(comm->reduce_scatter(dkv, P(m.bs.dkv_loc), static_cast<size_t>(S) * KV, s));
                RT_CUDA(cudaMemcpy2DAsync(dqkv + k.nq_l * D, static_cast<size_t>(Q) * 2, P(m.bs.dkv_loc),
                                          static_cast<size_t>(KV) * 2, static_cast<size_t>(KV) * 2, S,
                                          cudaMemcpyDeviceToDevice, s));
                return dh_rope(dqkv, Q, S, k.nq_l, k.nkv_l, D, k.rope_theta, k.cp_rank * S, 1, s);
            }
            RT_TRY(dh_attn_bwd(qkv, qkv + k.nq_l * D, qkv + (k.nq_l + k.nkv_l) * D, Q, Q, P(sl.o), A,
                               m.ptr<float>(sl.lse), P(m.bs.d_o), dqkv, dqkv + k.nq_l * D,
                               dqkv + (k.nq_l + k.nkv_l) * D, Q, Q, m.ptr<float>(m.bs.attn_scratch),
                               S, k.nq_l, k.nkv_l, D, scale, s));
            return dh_rope(dqkv, Q, S, k.nq_l, k.nkv_l, D, k.rope_theta, 0, 1, s);
        }
        case 35:  // qkv_dgrad
            return gemm(P(m.bs.dqkv), Q, false, W + p.wqkv, H, true,
                        tp1 ? P(m.bs.rs_out) : P(m.bs.dx_part), H, false, S, H, Q, false, cap, s);
        case 36:  // qkv_wgrad: dWqkv[Q,H] += dqkv^T ln0
            return gemm(P(m.bs.dqkv), Q, true, P(sl.ln0_full), H, true, G + p.wqkv, H, true, Q, H, S,
                        true, cap, s);
        case 37:  // ag0_bwd_rs
            RT_TRY(need_comm());
            return comm->reduce_scatter(P(m.bs.dx_part), P(m.bs.rs_out), TH, s);
        case 38:  // ln0_bwd (+ join of the attention-block skip gradient d_x1)
            return dh_rmsnorm_bwd(x_in, W + p.g0, m.ptr<float>(sl.rstd0), P(m.bs.rs_out), P(m.bs.d_x1), d_x,
                                  G + p.g0, m.ptr<float>(m.bs.ln_partial), T, H, s);
        case kSendAct:  // output of this visit's last layer -> next stage
            return m.ctx->pp ? m.ctx->pp->send(P(m.slots[op.slot].out), TH * 2, op.peer, xfer_tag(op), s)
                             : set_error(DH_ERR_CONFIG, "pipeline transfer without a stage group");
        case kRecvAct:  // input of this visit's first layer
            return m.ctx->pp ? m.ctx->pp->recv(k.split > 0 && op.layer == k.split ? P(m.mid_in[op.strand])
                                                                                 : P(m.mb_in[op.strand]),
                                               TH * 2, op.peer, xfer_tag(op), s)
                             : set_error(DH_ERR_CONFIG, "pipeline transfer without a stage group");
        case kSendGrad:  // input gradient of this visit's lowest layer -> previous stage
            return m.ctx->pp ? m.ctx->pp->send(d_x, TH * 2, op.peer, xfer_tag(op), s)
                             : set_error(DH_ERR_CONFIG, "pipeline transfer without a stage group");
        case kRecvGrad:  // dL/d(output) of this visit's top layer
            return m.ctx->pp ? m.ctx->pp->recv(op.layer == L - 1 ? P(m.mb_dy[op.strand]) : P(m.mid_dy[op.strand]),
                                               TH * 2, op.peer, xfer_tag(op), s)
                             : set_error(DH_ERR_CONFIG, "pipeline transfer without a stage group");
        case kOptNode: {  // AdamW of this layer's matrices (wqkv .. wd are contiguous)
            const size_t lo = p.wqkv, hi = op.layer + 1 < L ? m.lp[op.layer + 1].wqkv : m.n_params;
            return dh_adamw_dev(m.ptr<float>(m.w_master) + lo, W + lo, G + lo, m.ptr<float>(m.adam_m) + lo,
                                m.ptr<float>(m.adam_v) + lo, static_cast<long long>(hi - lo),
                                m.ptr<float>(m.opt_hp), s);
        }
        default:
            return set_error(DH_ERR_CONFIG, "launch_node: unknown template node " + std::to_string(node));
    }
}

int run_optimizer(Model& m, const dh_optim_cfg* oc, cudaStream_t s) {
    const ModelCfg& k = m.cfg;
    if (k.tp > 1 && m.ctx->comm) {
        // LayerNorm gammas are replicated across the TP group but see only
        // their sequence shard: sum their gradients (Megatron SP rule).
        RT_TRY(m.ctx->comm->all_reduce_f32(m.ptr<float>(m.w_grad), m.gamma_elems, s));
    }
    if (k.cp > 1 && m.ctx->comm) {
        // context parallelism: every weight is replicated over the CP group and
        // saw only this rank's tokens: sum the gradients (Megatron CP rule)
        RT_TRY(m.ctx->comm->all_reduce_f32(m.ptr<float>(m.w_grad), m.n_params, s));
    }
    if (k.moe && k.ep > 1 && m.ctx->comm) {
        // data-parallel replicas (gammas, attention, router): sum over the EP group
        float* g = m.ptr<float>(m.w_grad);
        RT_TRY(m.ctx->comm->all_reduce_f32(g, m.gamma_elems, s));
        for (const auto& p : m.lp) RT_TRY(m.ctx->comm->all_reduce_f32(g + p.wqkv, p.wg - p.wqkv, s));
    }
    if (!oc || !oc->enabled) return DH_OK;
    // with the per-layer AdamW ops in the program only the gammas remain
    const bool fused = m.fuse_optimizer && m.prog_has_opt;
    const long long n = static_cast<long long>(fused ? m.gamma_elems : m.n_params);
    RT_TRY(dh_adamw(m.ptr<float>(m.w_master), m.ptr(m.w_bf16), m.ptr<float>(m.w_grad), m.ptr<float>(m.adam_m),
                    m.ptr<float>(m.adam_v), n, oc->lr, oc->beta1, oc->beta2, oc->eps, oc->weight_decay,
                    m.adam_step, 1.f / (k.micro_batches * (k.moe ? k.ep : 1)), 1, s));
    if (fused) {  // disarm: a later bare program replay must not update the weights
        dh_adamw_hparams off{};
        RT_TRY(dh_adamw_set_hparams(m.ptr<float>(m.opt_hp), &off, s));
    }
    return DH_OK;
}

// Arms the in-program AdamW ops for this step (before the program runs).
int arm_optimizer(Model& m, const dh_optim_cfg* oc, cudaStream_t s) {
    if (!oc || !oc->enabled) return DH_OK;
    ++m.adam_step;
    if (!(m.fuse_optimizer && m.prog_has_opt)) return DH_OK;
    dh_adamw_hparams hp{};
    hp.lr = oc->lr;
    hp.beta1 = oc->beta1;
    hp.beta2 = oc->beta2;
    hp.eps = oc->eps;
    hp.weight_decay = oc->weight_decay;
    hp.bc1 = 1.f - std::pow(oc->beta1, static_cast<float>(m.adam_step));  // as dh_adamw
    hp.bc2 = 1.f - std::pow(oc->beta2, static_cast<float>(m.adam_step));
    hp.grad_scale = 1.f / (m.cfg.micro_batches * (m.cfg.moe ? m.cfg.ep : 1));
    hp.enabled = 1;
    return dh_adamw_set_hparams(m.ptr<float>(m.opt_hp), &hp, s);
}

}  // namespace dh
