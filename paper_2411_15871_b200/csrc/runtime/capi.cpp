// extern "C" face of the runtime (include/dh_capi.h, "runtime" section).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "nlohmann/json.hpp"
#include "runtime.hpp"

using nlohmann::json;

namespace dh {

// Kernels this repo launches for one node (NCCL kernels and memcpys excluded).
namespace {
int dense_kernels(const Model& m, int node, int layer);
}

int kernels_per_node(const Model& m, int node, int layer) {
    if (m.cfg.moe && node < kOptNode) {
        const int el = m.cfg.e_loc;
        switch (node) {
            case 15: case 21: case 28: return 1;
            case 10: return 2;                      // assign + gather
            case 13: case 23: case 24: return el;   // one GEMM per local expert
            case 12: case 25: case 26: return 2 * el;
            case 9: return 2;                       // logits GEMM + softmax/top-k
            case 29: return 3;                      // dlogits, dx GEMM, dwr GEMM
            case 11: case 14: case 22: case 27: return 0;  // all-to-all (NCCL / copies)
            default: {
                const int d = moe_dense_id(node);
                return d < 0 ? 0 : dense_kernels(m, d, layer);
            }
        }
    }
    return dense_kernels(m, node, layer);
}

namespace {
int dense_kernels(const Model& m, int node, int layer) {
    const bool group = m.cfg.nq_l != m.cfg.nkv_l;
    switch (node) {
        case 10: case 11: {  // (+ standalone SwiGLU on the later of the two when not in its epilogue)
            if (m.swiglu_in_epilogue) return 1;
            const auto& fs = m.plan.fwd_seq;
            const auto pos = [&](int id) { return std::find(fs.begin(), fs.end(), id) - fs.begin(); };
            return pos(node) > pos(node == 10 ? 11 : 10) ? 2 : 1;
        }
        case 22:
            return m.swiglu_in_epilogue ? 1 : 2;
        case 0: case 5: case 7: case 12: case 23: case 24: case 25:
        case 31: case 32: case 35: case 36:
            return 1;
        case 2: case 26: case 28: case 38:
            return 2;
        case kOptNode:
            return 1;
        case kSendAct: case kRecvAct: case kSendGrad: case kRecvGrad:
            return 0;  // staged device copies
        case 4:  // attn (+ KV-split combine when the launcher splits rows)
            return dh_attn_fwd_scratch_floats(m.cfg.seq, m.cfg.nq_l, m.cfg.nkv_l, m.cfg.head_dim) > 0 ? 2 : 1;
        case 14:
            return layer == m.cfg.layers - 1 ? 3 : 1;
        case 34:
            // dot, dK/dV + dQ (one tcgen05 launch), [group reduce], rope
            return 3 + (group ? 1 : 0);
        default:
            return 0;  // collectives (NCCL / loopback copies) and memcpy pass-throughs
    }
}
}  // namespace

}  // namespace dh

namespace {

weft::BestPlan trivial_plan(const dh::Model& m) {
    weft::BestPlan p;
    p.fwd_seq = weft::enumerate_topological_orders(m.fwd_dag, 1).at(0);
    p.bwd_seq = weft::enumerate_topological_orders(m.bwd_dag, 1).at(0);
    p.fwd_segmentation = {p.fwd_seq, {}};
    p.bwd_segmentation = {p.bwd_seq, {}};
    weft::PairStep st;
    st.fwd_seg = 1;
    st.bwd_seg = 1;
    p.plan.steps.push_back(st);
    return p;
}

struct TensorRef {
    void* ptr = nullptr;
    long long numel = 0;
    int dtype = 0;
};

int find_tensor(dh::Model& m, const std::string& name, int layer, int strand, TensorRef* r) {
    const auto& k = m.cfg;
    const long long H = k.hidden, S = k.seq, T = k.tok_loc, Q = k.qkv_n, A = k.attn_n, F = k.ffn_l;
    const int L = k.layers;
    auto bad = [&](const char* why) { return dh::set_error(DH_ERR_INVALID, std::string("tensor '") + name + "': " + why); };
    if (name == "x_in" || name == "dy") {
        if (strand < 0 || strand >= k.micro_batches) return bad("strand out of range");
        r->ptr = m.ptr(name == "x_in" ? m.mb_in[strand] : m.mb_dy[strand]);
        r->numel = T * H;
        return DH_OK;
    }
    if (name == "loss") {
        r->ptr = m.ptr(m.loss);
        r->numel = k.micro_batches;
        r->dtype = 1;
        return DH_OK;
    }
    if (name == "dx") {  // layer-0 input gradient of the most recent backward strand
        r->ptr = m.ptr(m.bs.grad[(L - 1) & 1]);
        r->numel = T * H;
        return DH_OK;
    }
    if (name == "y") {
        if (m.y_slot.empty() || strand < 0 || strand >= k.micro_batches) return bad("no program / strand");
        r->ptr = m.ptr(m.slots[m.y_slot[strand]].out);
        r->numel = T * H;
        return DH_OK;
    }
    const auto dot = name.find('.');
    if (dot == std::string::npos) return bad("unknown name");
    const std::string kind = name.substr(0, dot), t = name.substr(dot + 1);
    if (layer < 0 || layer >= L) return bad("layer out of range");
    const auto& p = m.lp[layer];
    size_t off = 0;
    long long n = 0;
    if (t == "g0") off = p.g0, n = H;
    else if (t == "g1") off = p.g1, n = H;
    else if (t == "wqkv") off = p.wqkv, n = Q * H;
    else if (t == "wo") off = p.wo, n = H * A;
    else if (t == "wg") off = p.wg, n = F * H;
    else if (t == "wu") off = p.wu, n = F * H;
    else if (t == "wd") off = p.wd, n = H * F;
    // MoE: router [E,H]; stacked local experts w1g / w1u [e_loc,F,H], w2 [e_loc,H,F]
    else if (k.moe && t == "wr") off = p.wr, n = static_cast<long long>(k.experts) * H;
    else if (k.moe && t == "w1g") off = p.wg, n = static_cast<long long>(k.e_loc) * F * H;
    else if (k.moe && t == "w1u") off = p.wu, n = static_cast<long long>(k.e_loc) * F * H;
    else if (k.moe && t == "w2") off = p.wd, n = static_cast<long long>(k.e_loc) * H * F;
    else if (kind != "act") return bad("unknown parameter");
    if (kind == "w") {
        r->ptr = m.ptr<char>(m.w_bf16) + off * 2;
        r->numel = n;
        return DH_OK;
    }
    if (kind == "grad" || kind == "master") {
        r->ptr = m.ptr<char>(kind == "grad" ? m.w_grad : m.w_master) + off * 4;
        r->numel = n;
        r->dtype = 1;
        return DH_OK;
    }
    if (kind == "act") {
        // saved activations of (strand, layer) as placed by the current program
        // (valid until the slot is reused; with micro_batches == 1 after a step).
        if (m.prog.ops.empty()) return bad("no program");
        int slot = -1;
        for (const auto& o : m.prog.ops) {
            if (o.strand == strand && o.layer == layer) {
                slot = o.slot;
                break;
            }
        }
        if (slot < 0) return bad("no such (strand, layer)");
        const dh::Slot& s = m.slots[slot];
        const std::pair<const char*, std::pair<const dh::Buf*, int>> fields[] = {
            {"out", {&s.out, 0}},       {"rstd0", {&s.rstd0, 1}}, {"ln0_full", {&s.ln0_full, 0}},
            {"qkv", {&s.qkv, 0}},       {"o", {&s.o, 0}},         {"lse", {&s.lse, 1}},
            {"x1", {&s.x1, 0}},         {"rstd1", {&s.rstd1, 1}}, {"ln1_full", {&s.ln1_full, 0}},
            {"gate", {&s.gate, 0}},     {"up", {&s.up, 0}},       {"act", {&s.act, 0}},
            {"probs", {&s.probs, 1}},   {"wts", {&s.wts, 1}},     {"ids", {&s.ids, 1}},
            {"mslot", {&s.mslot, 1}},   {"slot_src", {&s.slot_src, 1}}, {"xe", {&s.xe, 0}},
            {"y_moe", {&s.y, 0}}};
        for (const auto& [fname, bd] : fields) {
            if (t == fname) {
                r->ptr = m.ptr(*bd.first);
                r->dtype = bd.second;
                r->numel = static_cast<long long>(bd.first->bytes / (bd.second ? 4 : 2));
                return DH_OK;
            }
        }
        return bad("unknown activation field");
    }
    (void)S;
    return bad("unknown kind");
}

}  // namespace

namespace dh {

int configure_plan(Model& mm, const char* plan_json, const char* profile_json,
                   const char* cluster_json) {
    Model* m = &mm;
    try {
        m->solo_us.clear();
        m->plan_overlap = weft::OverlapTable{};
        weft::Profile prof;
        if (profile_json && *profile_json) {
            prof = weft::parse_profile(profile_json);
            m->plan_overlap = prof.overlap;
        }
        if (cluster_json && *cluster_json) {
            const json c = json::parse(cluster_json);
            weft::ClusterSpec cl;
            cl.name = c.value("name", std::string("custom"));
            cl.gpus = c.at("gpus").get<int>();
            cl.per_node = c.at("per_node").get<int>();
            cl.peak_tflops = c.at("peak_tflops").get<double>();
            cl.local_bw_gbs = c.at("local_bw_gbs").get<double>();
            cl.cross_bw_gbs = c.at("cross_bw_gbs").get<double>();
            cl.mem_gb = c.at("mem_gb").get<double>();
            cl.bw_efficiency = c.value("bw_efficiency", 0.5);
            RT_TRY(build_dags(*m, cl, &prof.solo));
        }
        for (const auto* dag : {&m->fwd_dag, &m->bwd_dag}) {
            for (const auto& n : dag->nodes) {
                if (auto t = prof.solo.get(n.cls, n.name)) m->solo_us[n.id] = *t;
            }
        }
        if (plan_json && *plan_json) {
            m->plan = weft::parse_plan_json(plan_json);
            if (!weft::validate_sequence(m->fwd_dag, m->plan.fwd_seq) ||
                !weft::validate_sequence(m->bwd_dag, m->plan.bwd_seq)) {
                return set_error(DH_ERR_CONFIG,
                                 "plan sequences are not valid orders of this model's layer DAG "
                                 "(plan built for a different tp / template?)");
            }
        } else {
            m->plan = trivial_plan(*m);
        }
        m->have_plan = true;
    } catch (const std::exception& e) {
        return set_error(DH_ERR_CONFIG, e.what());
    }
    return DH_OK;
}

}  // namespace dh

extern "C" {

int dh_model_create(dh_ctx* ctx, const dh_model_cfg* cfg, dh_model** out) {
    if (!ctx || !cfg || !out) return dh::set_error(DH_ERR_INVALID, "dh_model_create: null argument");
    dh::Model* m = nullptr;
    const int rc = dh::model_create(ctx, cfg, &m);
    if (rc != DH_OK) return rc;
    *out = static_cast<dh_model*>(m);
    return DH_OK;
}

int dh_model_destroy(dh_model* m) {
    dh::model_destroy(m);
    return DH_OK;
}

int dh_model_set_plan(dh_model* m, const char* plan_json, const char* profile_json,
                      const char* cluster_json, int mode) {
    if (!m) return dh::set_error(DH_ERR_INVALID, "null model");
    if (mode < 0 || mode > 4)
        return dh::set_error(DH_ERR_INVALID,
                             "mode must be 0 (SI), 1 (sequential), 2 (SI, relaxed steps), 3 (W pipeline stage) "
                             "or 4 (SI, relaxed steps, deferred attention weight gradients)");
    if (mode == 3 && m->cfg.pp_size != m->ctx->pp_size)
        return dh::set_error(DH_ERR_CONFIG, "w_pipeline: dh_model_cfg.pp_size differs from the context's stage group");
    RT_TRY(dh::configure_plan(*m, plan_json, profile_json, cluster_json));
    return dh::lower_program(*m, mode);
}

int dh_lower_json(const dh_model_cfg* cfg, int tp, int rank, const char* plan_json,
                  const char* profile_json, int mode, char** out) {
    if (!cfg || !out) return dh::set_error(DH_ERR_INVALID, "null argument");
    if (mode < 0 || mode > 4)
        return dh::set_error(DH_ERR_INVALID,
                             "mode must be 0 (SI), 1 (sequential), 2 (SI, relaxed steps), 3 (W pipeline stage) "
                             "or 4 (SI, relaxed steps, deferred attention weight gradients)");
    dh::Model m;  // host-only: no context, no pool
    RT_TRY(dh::derive_cfg(cfg, tp, rank, &m.cfg));
    RT_TRY(dh::build_dags(m, dh::default_cluster(), nullptr));
    RT_TRY(dh::configure_plan(m, plan_json, profile_json, nullptr));
    RT_TRY(dh::lower_ops(m, mode));
    json ops = json::array();
    for (const auto& o : m.prog.ops) {
        ops.push_back({{"strand", o.strand}, {"layer", o.layer}, {"node", o.node}, {"lane", o.lane},
                       {"slot", o.slot}, {"prev_slot", o.prev_slot}, {"first_dx", o.first_dx},
                       {"peer", o.peer}, {"part", o.part}, {"waits", o.waits}});
    }
    json j = {{"ops", ops}, {"slots", m.cfg.slots > 0 ? m.cfg.slots : m.cfg.layers + 1},
              {"peak_slots", m.peak_slots}, {"fwd_seq", m.plan.fwd_seq},
              {"bwd_seq", m.plan.bwd_seq}, {"mode", mode}};
    const std::string s = j.dump();
    *out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*out, s.c_str(), s.size() + 1);
    return DH_OK;
}

int dh_model_set_fuse_optimizer(dh_model* m, int on) {
    if (!m) return dh::set_error(DH_ERR_INVALID, "null model");
    m->fuse_optimizer = on != 0;
    return DH_OK;
}

int dh_model_set_overlap_ctas(dh_model* m, int gemm_ctas) {
    if (!m) return dh::set_error(DH_ERR_INVALID, "null model");
    m->gemm_ctas_overlap = gemm_ctas;
    if (m->graph) {
        cudaGraphExecDestroy(m->graph);
        m->graph = nullptr;
    }
    return DH_OK;
}

int dh_model_run_program(dh_model* m, int use_graph) {
    if (!m) return dh::set_error(DH_ERR_INVALID, "null model");
    return dh::run_program(*m, use_graph != 0);
}

int dh_model_step(dh_model* m, const dh_optim_cfg* optim, int use_graph) {
    if (!m) return dh::set_error(DH_ERR_INVALID, "null model");
    RT_TRY(dh::arm_optimizer(*m, optim, m->ctx->lane[0]));
    RT_TRY(dh::run_program(*m, use_graph != 0));
    return dh::run_optimizer(*m, optim, m->ctx->lane[0]);
}

int dh_model_zero_grads(dh_model* m) {
    if (!m) return dh::set_error(DH_ERR_INVALID, "null model");
    RT_CUDA(cudaSetDevice(m->ctx->device));
    RT_CUDA(cudaMemsetAsync(m->ptr(m->w_grad), 0, m->w_grad.bytes, m->ctx->lane[0]));
    return DH_OK;
}

int dh_model_sync(dh_model* m) {
    if (!m) return dh::set_error(DH_ERR_INVALID, "null model");
    RT_CUDA(cudaSetDevice(m->ctx->device));
    for (auto s : m->ctx->lane) RT_CUDA(cudaStreamSynchronize(s));
    if (m->ctx->pp) RT_TRY(m->ctx->pp->sync());
    return DH_OK;
}

int dh_model_tensor(dh_model* m, const char* name, int layer, int strand, void** ptr,
                    long long* numel, int* dtype) {
    if (!m || !name) return dh::set_error(DH_ERR_INVALID, "null argument");
    TensorRef r;
    RT_TRY(find_tensor(*m, name, layer, strand, &r));
    if (ptr) *ptr = r.ptr;
    if (numel) *numel = r.numel;
    if (dtype) *dtype = r.dtype;
    return DH_OK;
}

int dh_model_info_json(dh_model* m, char** out) {
    if (!m || !out) return dh::set_error(DH_ERR_INVALID, "null argument");
    const auto& k = m->cfg;
    json j;
    j["pool_bytes"] = m->pool_bytes;
    j["usage"] = m->usage;
    j["n_params"] = m->n_params;
    j["slots"] = m->slots.size();
    size_t slot_bytes = 0;
    if (!m->slots.empty()) {
        const dh::Slot& s = m->slots[0];
        for (const dh::Buf* b : {&s.out, &s.rstd0, &s.ln0_full, &s.qkv, &s.o, &s.lse, &s.x1,
                                 &s.rstd1, &s.ln1_full, &s.gate, &s.up, &s.act})
            slot_bytes += (b->bytes + 255) & ~static_cast<size_t>(255);
    }
    j["slot_bytes"] = slot_bytes;
    j["cfg"] = {{"hidden", k.hidden}, {"ffn", k.ffn}, {"n_heads", k.n_heads}, {"n_kv_heads", k.n_kv_heads},
                {"head_dim", k.head_dim}, {"layers", k.layers}, {"seq", k.seq}, {"tp", k.tp},
                {"rank", k.rank}, {"micro_batches", k.micro_batches}};
    int launches = 0;
    std::array<int, dh::kLanes> per_lane{};
    json ops = json::array();
    for (const auto& o : m->prog.ops) {
        launches += dh::kernels_per_node(*m, o.node, o.layer);
        per_lane[o.lane]++;
        if (ops.size() < 4096) ops.push_back({o.strand, o.layer, o.node, o.lane, o.slot, o.waits});
    }
    j["program"] = {{"mode", m->prog.mode}, {"ops", m->prog.ops.size()}, {"ops_per_lane", per_lane},
                    {"kernel_launches", launches + 1 /*adamw*/}, {"list", ops},
                    {"fwd_seq", m->plan.fwd_seq}, {"bwd_seq", m->plan.bwd_seq},
                    {"comm", m->ctx->comm ? m->ctx->comm->name() : "none"}};
    const std::string s = j.dump();
    *out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*out, s.c_str(), s.size() + 1);
    return DH_OK;
}

void dh_free_string(char* s) { std::free(s); }

int dh_model_set_skip_comm(dh_model* m, int skip) {
    if (!m) return dh::set_error(DH_ERR_INVALID, "null model");
    m->skip_comm = skip != 0;
    if (!m->have_plan) return DH_OK;
    return dh::lower_program(*m, m->prog.mode);  // re-lower without / with collectives
}

int dh_model_probe(dh_model* m, int node) {
    if (!m) return dh::set_error(DH_ERR_INVALID, "null model");
    return dh::set_probe(*m, node);
}

int dh_model_probe_read(dh_model* m, double* total_ms, int* count) {
    if (!m || !total_ms || !count) return dh::set_error(DH_ERR_INVALID, "null argument");
    return dh::read_probe(*m, -1, total_ms, count);
}

int dh_model_probe_read_node(dh_model* m, int node, double* total_ms, int* count) {
    if (!m || !total_ms || !count) return dh::set_error(DH_ERR_INVALID, "null argument");
    return dh::read_probe(*m, node, total_ms, count);
}

}  // extern "C"
