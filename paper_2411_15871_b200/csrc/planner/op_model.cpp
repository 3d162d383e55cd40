// L2 operator model: layer templates, roofline instantiation, linearisations.
//
// Behaviour follows /root/reference/proj/src/op_model.cpp:
//   LayerDag::validate (Kahn)            :25-62
//   builtin templates dense_tp_sp/moe_ep :74-171  (restated here as a table)
//   node_cost                            :250-310 (fp64 expression order kept)
//   build_layer_dag_from                 :314-404
//   enumerate_topological_orders         :416-456
//   validate_sequence                    :458-471
#include "weft/op_model.hpp"

#include <algorithm>
#include <functional>
#include <fstream>
#include <map>
#include <set>
#include <sstream>

#include "nlohmann/json.hpp"
#include "weft/overlap_profile.hpp"

namespace weft {

using nlohmann::json;

const OpNode* LayerDag::find(int id) const {
    auto it = std::find_if(nodes.begin(), nodes.end(), [id](const OpNode& n) { return n.id == id; });
    return it == nodes.end() ? nullptr : &*it;
}

void LayerDag::validate() const {
    std::map<int, int> indeg;  // ordered: the ready stack starts in id order
    for (const auto& n : nodes) {
        if (!indeg.emplace(n.id, 0).second) {
            throw ConfigError("duplicate node id " + std::to_string(n.id));
        }
    }
    std::map<int, std::vector<int>> succ;
    for (const auto& e : edges) {
        if (!indeg.count(e.first) || !indeg.count(e.second)) {
            throw ConfigError("edge references missing node: " + std::to_string(e.first) + "->" +
                              std::to_string(e.second));
        }
    }
    for (const auto& e : edges) {
        succ[e.first].push_back(e.second);
        indeg[e.second] += 1;
    }
    std::vector<int> stack;
    for (const auto& [id, d] : indeg) {
        if (d == 0) stack.push_back(id);
    }
    std::size_t popped = 0;
    while (!stack.empty()) {
        const int id = stack.back();
        stack.pop_back();
        ++popped;
        for (int c : succ[id]) {
            if (--indeg[c] == 0) stack.push_back(c);
        }
    }
    if (popped != nodes.size()) throw ConfigError("layer dag contains a cycle");
}

// ---------------------------------------------------------------------------
// Builtin templates (data). Node ids, names, classes, requirement tags and
// edges are the reference's dense_tp_sp / moe_ep graphs.

namespace {

struct TNode {
    int id;
    const char* name;
    const char* cls;
    bool fwd;
    const char* req;  // "" when unconditional
};

constexpr TNode kDenseNodes[] = {
    {0, "ln0", "LayerNorm", true, ""},
    {1, "ag0", "AllGather", true, "tp_sp"},
    {2, "qkv", "GEMM", true, ""},
    {3, "cp_kv_exchange", "SendRecv", true, "cp"},
    {4, "attn", "FlashAttention", true, ""},
    {5, "attn_proj", "GEMM", true, ""},
    {6, "rs0", "ReduceScatter", true, "tp_sp"},
    {7, "bda0", "FusedBDA", true, ""},
    {8, "ln1", "LayerNorm", true, ""},
    {9, "ag1", "AllGather", true, "tp_sp"},
    {10, "mlp_gate", "GEMM", true, ""},
    {11, "mlp_up", "GEMM", true, ""},
    {12, "mlp_down", "GEMM", true, ""},
    {13, "rs1", "ReduceScatter", true, "tp_sp"},
    {14, "bda1", "FusedBDA", true, ""},
    {20, "bda1_bwd", "FusedBDA", false, ""},
    {21, "rs1_bwd_ag", "AllGather", false, "tp_sp"},
    {22, "mlp_down_dgrad", "GEMM", false, ""},
    {23, "mlp_down_wgrad", "WeightGrad", false, ""},
    {24, "mlp_gate_dgrad", "GEMM", false, ""},
    {25, "mlp_up_dgrad", "GEMM", false, ""},
    {26, "mlp_fc1_wgrad", "WeightGrad", false, ""},
    {27, "ag1_bwd_rs", "ReduceScatter", false, "tp_sp"},
    {28, "ln1_bwd", "LayerNorm", false, ""},
    {29, "bda0_bwd", "FusedBDA", false, ""},
    {30, "rs0_bwd_ag", "AllGather", false, "tp_sp"},
    {31, "attn_proj_dgrad", "GEMM", false, ""},
    {32, "attn_proj_wgrad", "WeightGrad", false, ""},
    {33, "cp_kv_exchange_bwd", "SendRecv", false, "cp"},
    {34, "attn_bwd", "FlashAttentionBwd", false, ""},
    {35, "qkv_dgrad", "GEMM", false, ""},
    {36, "qkv_wgrad", "WeightGrad", false, ""},
    {37, "ag0_bwd_rs", "ReduceScatter", false, "tp_sp"},
    {38, "ln0_bwd", "LayerNorm", false, ""},
};

constexpr int kDenseEdges[][2] = {
    {0, 1},   {1, 2},   {2, 3},   {3, 4},   {4, 5},   {5, 6},   {6, 7},   {7, 8},   {8, 9},
    {9, 10},  {9, 11},  {10, 12}, {11, 12}, {12, 13}, {13, 14}, {20, 21}, {21, 22}, {21, 23},
    {22, 24}, {22, 25}, {22, 26}, {24, 27}, {25, 27}, {27, 28}, {28, 29}, {29, 30}, {30, 31},
    {30, 32}, {31, 33}, {33, 34}, {34, 35}, {34, 36}, {35, 37}, {37, 38},
};

constexpr TNode kMoeNodes[] = {
    {0, "ln0", "LayerNorm", true, ""},
    {1, "ag0", "AllGather", true, "tp_sp"},
    {2, "qkv", "GEMM", true, ""},
    {3, "cp_kv_exchange", "SendRecv", true, "cp"},
    {4, "attn", "FlashAttention", true, ""},
    {5, "attn_proj", "GEMM", true, ""},
    {6, "rs0", "ReduceScatter", true, "tp_sp"},
    {7, "bda0", "FusedBDA", true, ""},
    {8, "ln1", "LayerNorm", true, ""},
    {9, "router", "Router", true, ""},
    {10, "permute", "Permute", true, ""},
    {11, "a2a_dispatch", "AllToAll", true, "ep"},
    {12, "expert_fc1", "GroupGEMM", true, ""},
    {13, "expert_fc2", "GroupGEMM", true, ""},
    {14, "a2a_combine", "AllToAll", true, "ep"},
    {15, "unpermute", "Permute", true, ""},
    {16, "bda1", "FusedBDA", true, ""},
    {20, "bda1_bwd", "FusedBDA", false, ""},
    {21, "unpermute_bwd", "Permute", false, ""},
    {22, "a2a_combine_bwd", "AllToAll", false, "ep"},
    {23, "expert_fc2_dgrad", "GroupGEMM", false, ""},
    {24, "expert_fc2_wgrad", "WeightGrad", false, ""},
    {25, "expert_fc1_dgrad", "GroupGEMM", false, ""},
    {26, "expert_fc1_wgrad", "WeightGrad", false, ""},
    {27, "a2a_dispatch_bwd", "AllToAll", false, "ep"},
    {28, "permute_bwd", "Permute", false, ""},
    {29, "router_bwd", "Router", false, ""},
    {30, "ln1_bwd", "LayerNorm", false, ""},
    {31, "bda0_bwd", "FusedBDA", false, ""},
    {32, "rs0_bwd_ag", "AllGather", false, "tp_sp"},
    {33, "attn_proj_dgrad", "GEMM", false, ""},
    {34, "attn_proj_wgrad", "WeightGrad", false, ""},
    {35, "cp_kv_exchange_bwd", "SendRecv", false, "cp"},
    {36, "attn_bwd", "FlashAttentionBwd", false, ""},
    {37, "qkv_dgrad", "GEMM", false, ""},
    {38, "qkv_wgrad", "WeightGrad", false, ""},
    {39, "ag0_bwd_rs", "ReduceScatter", false, "tp_sp"},
    {40, "ln0_bwd", "LayerNorm", false, ""},
};

constexpr int kMoeEdges[][2] = {
    {0, 1},   {1, 2},   {2, 3},   {3, 4},   {4, 5},   {5, 6},   {6, 7},   {7, 8},   {8, 9},
    {9, 10},  {10, 11}, {11, 12}, {12, 13}, {13, 14}, {14, 15}, {15, 16}, {20, 21}, {21, 22},
    {22, 23}, {22, 24}, {23, 25}, {23, 26}, {25, 27}, {27, 28}, {28, 29}, {29, 30}, {30, 31},
    {31, 32}, {32, 33}, {32, 34}, {33, 35}, {35, 36}, {36, 37}, {36, 38}, {37, 39}, {39, 40},
};

template <std::size_t NN, std::size_t NE>
json template_to_json(const char* name, const char* doc, const TNode (&nodes)[NN],
                      const int (&edges)[NE][2]) {
    json jt;
    jt["name"] = name;
    jt["doc"] = doc;
    jt["nodes"] = json::array();
    for (const auto& n : nodes) {
        json jn = {{"id", n.id}, {"name", n.name}, {"class", n.cls},
                   {"pass", n.fwd ? "forward" : "backward"}};
        if (n.req[0] != '\0') jn["requires"] = n.req;
        jt["nodes"].push_back(std::move(jn));
    }
    jt["edges"] = json::array();
    for (const auto& e : edges) jt["edges"].push_back({e[0], e[1]});
    return jt;
}

const std::string& builtin_json_text() {
    static const std::string text = [] {
        json j;
        j["templates"] = json::array();
        j["templates"].push_back(template_to_json(
            "dense_tp_sp",
            "Dense transformer layer under TP(+SP); tp_sp nodes need tp>1, cp nodes need cp>1.",
            kDenseNodes, kDenseEdges));
        j["templates"].push_back(template_to_json(
            "moe_ep",
            "MoE transformer layer under EP; ep nodes need ep>1, tp_sp nodes need tp>1, cp nodes "
            "need cp>1.",
            kMoeNodes, kMoeEdges));
        return j.dump(2) + "\n";
    }();
    return text;
}

DagTemplate template_from_json(const json& jt) {
    DagTemplate t;
    t.name = jt.at("name").get<std::string>();
    for (const auto& jn : jt.at("nodes")) {
        DagTemplate::Node n;
        n.id = jn.at("id").get<int>();
        n.name = jn.at("name").get<std::string>();
        n.cls = parse_operator_class(jn.at("class").get<std::string>());
        n.pass = parse_pass(jn.at("pass").get<std::string>());
        if (jn.contains("requires")) n.requires_dim = jn.at("requires").get<std::string>();
        t.nodes.push_back(std::move(n));
    }
    for (const auto& je : jt.at("edges")) {
        t.edges.emplace_back(je.at(0).get<int>(), je.at(1).get<int>());
    }
    return t;
}

const std::vector<DagTemplate>& builtin_templates() {
    static const std::vector<DagTemplate> all = parse_dag_templates(builtin_json_text());
    return all;
}

}  // namespace

std::vector<DagTemplate> parse_dag_templates(const std::string& json_text) {
    json doc;
    try {
        doc = json::parse(json_text);
    } catch (const json::exception& e) {
        throw ConfigError(std::string("dag template parse error: ") + e.what());
    }
    std::vector<DagTemplate> out;
    try {
        for (const auto& jt : doc.at("templates")) out.push_back(template_from_json(jt));
    } catch (const json::exception& e) {
        throw ConfigError(std::string("dag template schema error: ") + e.what());
    }
    return out;
}

std::vector<DagTemplate> load_dag_templates(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw ConfigError("cannot open dag template file: " + path);
    std::ostringstream buf;
    buf << f.rdbuf();
    return parse_dag_templates(buf.str());
}

const DagTemplate& builtin_template(const std::string& name) {
    for (const auto& t : builtin_templates()) {
        if (t.name == name) return t;
    }
    throw ConfigError("unknown builtin template: " + name);
}

std::string builtin_template_json() { return builtin_json_text(); }

// ---------------------------------------------------------------------------
// Roofline instantiation

namespace {

enum class CostKind {
    none, qkv, attn, attn_bwd, attn_proj, mlp_fc1, mlp_fc1_wgrad, mlp_down, norm, bda,
    router, permute, expert_fc1, expert_fc2, tp_collective, cp_exchange, ep_all_to_all,
};

CostKind cost_kind(const std::string& name) {
    static const std::map<std::string, CostKind> kKinds = {
        {"qkv", CostKind::qkv}, {"qkv_dgrad", CostKind::qkv}, {"qkv_wgrad", CostKind::qkv},
        {"attn", CostKind::attn}, {"attn_bwd", CostKind::attn_bwd},
        {"attn_proj", CostKind::attn_proj}, {"attn_proj_dgrad", CostKind::attn_proj},
        {"attn_proj_wgrad", CostKind::attn_proj},
        {"mlp_gate", CostKind::mlp_fc1}, {"mlp_up", CostKind::mlp_fc1},
        {"mlp_gate_dgrad", CostKind::mlp_fc1}, {"mlp_up_dgrad", CostKind::mlp_fc1},
        {"mlp_fc1_wgrad", CostKind::mlp_fc1_wgrad},
        {"mlp_down", CostKind::mlp_down}, {"mlp_down_dgrad", CostKind::mlp_down},
        {"mlp_down_wgrad", CostKind::mlp_down},
        {"ln0", CostKind::norm}, {"ln1", CostKind::norm}, {"ln0_bwd", CostKind::norm},
        {"ln1_bwd", CostKind::norm},
        {"bda0", CostKind::bda}, {"bda1", CostKind::bda}, {"bda0_bwd", CostKind::bda},
        {"bda1_bwd", CostKind::bda},
        {"router", CostKind::router}, {"router_bwd", CostKind::router},
        {"permute", CostKind::permute}, {"unpermute", CostKind::permute},
        {"permute_bwd", CostKind::permute}, {"unpermute_bwd", CostKind::permute},
        {"expert_fc1", CostKind::expert_fc1}, {"expert_fc1_dgrad", CostKind::expert_fc1},
        {"expert_fc1_wgrad", CostKind::expert_fc1},
        {"expert_fc2", CostKind::expert_fc2}, {"expert_fc2_dgrad", CostKind::expert_fc2},
        {"expert_fc2_wgrad", CostKind::expert_fc2},
        {"ag0", CostKind::tp_collective}, {"ag1", CostKind::tp_collective},
        {"rs0", CostKind::tp_collective}, {"rs1", CostKind::tp_collective},
        {"rs1_bwd_ag", CostKind::tp_collective}, {"ag1_bwd_rs", CostKind::tp_collective},
        {"rs0_bwd_ag", CostKind::tp_collective}, {"ag0_bwd_rs", CostKind::tp_collective},
        {"cp_kv_exchange", CostKind::cp_exchange}, {"cp_kv_exchange_bwd", CostKind::cp_exchange},
        {"a2a_dispatch", CostKind::ep_all_to_all}, {"a2a_combine", CostKind::ep_all_to_all},
        {"a2a_dispatch_bwd", CostKind::ep_all_to_all}, {"a2a_combine_bwd", CostKind::ep_all_to_all},
    };
    auto it = kKinds.find(name);
    return it == kKinds.end() ? CostKind::none : it->second;
}

struct NodeWork {
    double flops = 0.0;
    std::int64_t wire = 0;
    int extent = 1;  // ranks spanned by the communication group (tp innermost)
};

constexpr double kBytesPerElem = 2.0;  // bf16 on the wire

// Every expression keeps the reference's left-to-right evaluation order so the
// fp64 results (and therefore every derived duration) are bit-identical.
NodeWork node_work(const std::string& name, const ModelSpec& m, const ParallelismSpec& p) {
    const double tokens = static_cast<double>(m.seq_len) / p.cp;
    const double h = m.hidden, f = m.intermediate, s = m.seq_len;
    const double tp = p.tp, ep = p.ep;
    const double topk = m.topk.value_or(1);
    const auto mm = [](double a, double k, double n) { return 2.0 * a * k * n; };

    NodeWork w;
    switch (cost_kind(name)) {
        case CostKind::qkv: w.flops = mm(tokens, h, 3.0 * h / tp); break;
        case CostKind::attn: w.flops = 2.0 * tokens * s * h / tp; break;
        case CostKind::attn_bwd: w.flops = 2.5 * 2.0 * tokens * s * h / tp; break;
        case CostKind::attn_proj: w.flops = mm(tokens, h / tp, h); break;
        case CostKind::mlp_fc1: w.flops = mm(tokens, h, f / tp); break;
        case CostKind::mlp_fc1_wgrad: w.flops = mm(tokens, h, 2.0 * f / tp); break;
        case CostKind::mlp_down: w.flops = mm(tokens, f / tp, h); break;
        case CostKind::norm: w.flops = 10.0 * tokens * h / (p.sp ? tp : 1.0); break;
        case CostKind::bda: w.flops = 8.0 * tokens * h / (p.sp ? tp : 1.0); break;
        case CostKind::router: w.flops = 2.0 * tokens * h * m.experts.value_or(1); break;
        case CostKind::permute: w.flops = 2.0 * tokens * h * topk; break;
        case CostKind::expert_fc1: w.flops = mm(tokens * topk / ep, h, 2.0 * f / tp); break;
        case CostKind::expert_fc2: w.flops = mm(tokens * topk / ep, f / tp, h); break;
        case CostKind::tp_collective: {
            const double payload = tokens * h * kBytesPerElem;
            w.wire = static_cast<std::int64_t>(payload * (tp - 1.0) / tp);
            w.extent = p.tp;
            break;
        }
        case CostKind::cp_exchange:
            w.wire = static_cast<std::int64_t>(2.0 * tokens * (h / tp) * kBytesPerElem *
                                               (p.cp - 1.0));
            w.extent = p.tp * p.cp;
            break;
        case CostKind::ep_all_to_all: {
            const double payload = tokens * topk * h * kBytesPerElem;
            w.wire = static_cast<std::int64_t>(payload * (ep - 1.0) / ep);
            w.extent = p.tp * p.cp * p.ep;
            break;
        }
        case CostKind::none: break;
    }
    return w;
}

bool node_active(const DagTemplate& t, const DagTemplate::Node& n, const ParallelismSpec& p) {
    const std::string& r = n.requires_dim;
    if (r.empty()) return true;
    if (r == "tp_sp") return p.tp > 1;  // reference gates on tp only (op_model.cpp:327)
    if (r == "cp") return p.cp > 1;
    if (r == "ep") return p.ep > 1;
    throw ConfigError("template '" + t.name + "': unknown requires tag '" + r + "'");
}

}  // namespace

std::pair<LayerDag, LayerDag> build_layer_dag_from(const DagTemplate& tmpl, const ModelSpec& model,
                                                   const ParallelismSpec& par,
                                                   const ClusterSpec& cluster,
                                                   const SoloTimeTable* solo) {
    model.validate();
    par.validate();
    cluster.validate();
    if (par.ep > 1 && !model.is_moe()) {
        throw ConfigError("EP requested with non-MoE model '" + model.name + "'");
    }

    std::map<int, const DagTemplate::Node*> keep;
    for (const auto& n : tmpl.nodes) {
        if (node_active(tmpl, n, par)) keep[n.id] = &n;
    }
    // Contract every dropped node: connect each of its producers to each of
    // its consumers (in template order of removal).
    std::set<std::pair<int, int>> edge_set(tmpl.edges.begin(), tmpl.edges.end());
    for (const auto& n : tmpl.nodes) {
        if (keep.count(n.id)) continue;
        std::vector<int> into, outof;
        for (auto it = edge_set.begin(); it != edge_set.end();) {
            if (it->second == n.id) {
                into.push_back(it->first);
                it = edge_set.erase(it);
            } else if (it->first == n.id) {
                outof.push_back(it->second);
                it = edge_set.erase(it);
            } else {
                ++it;
            }
        }
        for (int a : into) {
            for (int b : outof) edge_set.emplace(a, b);
        }
    }

    std::pair<LayerDag, LayerDag> out;
    out.first.pass = Pass::forward;
    out.second.pass = Pass::backward;
    for (const auto& [id, tn] : keep) {
        const NodeWork w = node_work(tn->name, model, par);
        const bool local = w.extent <= cluster.per_node;
        OpNode op;
        op.id = id;
        op.cls = tn->cls;
        op.pass = tn->pass;
        op.name = tn->name;
        op.flops = w.flops;
        op.bytes = w.wire;
        op.lane = !is_comm_class(tn->cls) ? Lane::compute
                                          : (local ? Lane::local_comm : Lane::cross_comm);
        double t = 0.0;
        if (solo) {
            if (const auto hit = solo_lookup(*solo, tn->cls, tn->name)) t = *hit;
        }
        if (t <= 0.0) {
            if (op.lane == Lane::compute) {
                t = w.flops / (cluster.peak_tflops * 1e6);
            } else {
                const double bw = local ? cluster.local_bw_gbs : cluster.cross_bw_gbs;
                t = static_cast<double>(w.wire) / (bw * cluster.bw_efficiency * 1e3);
            }
        }
        op.duration_us = t;
        (tn->pass == Pass::forward ? out.first : out.second).nodes.push_back(std::move(op));
    }
    for (const auto& e : edge_set) {
        const Pass a = keep.at(e.first)->pass;
        if (a != keep.at(e.second)->pass) {
            throw ConfigError("template '" + tmpl.name + "': edge crosses passes");
        }
        (a == Pass::forward ? out.first : out.second).edges.push_back(e);
    }
    out.first.validate();
    out.second.validate();
    return out;
}

std::pair<LayerDag, LayerDag> build_layer_dag(const ModelSpec& model, const ParallelismSpec& par,
                                              const ClusterSpec& cluster,
                                              const SoloTimeTable* solo) {
    return build_layer_dag_from(builtin_template(model.is_moe() ? "moe_ep" : "dense_tp_sp"), model,
                                par, cluster, solo);
}

// ---------------------------------------------------------------------------
// Linearisations

std::vector<std::vector<int>> enumerate_topological_orders(const LayerDag& dag, std::size_t cap) {
    if (cap == 0) throw ConfigError("enumeration cap must be >= 1");
    dag.validate();

    // Dense index space over ascending ids.
    std::vector<int> ids;
    ids.reserve(dag.nodes.size());
    for (const auto& n : dag.nodes) ids.push_back(n.id);
    std::sort(ids.begin(), ids.end());
    const std::size_t n = ids.size();
    auto index_of = [&](int id) {
        return static_cast<std::size_t>(std::lower_bound(ids.begin(), ids.end(), id) - ids.begin());
    };
    std::vector<int> indeg(n, 0);
    std::vector<std::vector<std::size_t>> succ(n);
    for (const auto& [p, c] : dag.edges) {
        succ[index_of(p)].push_back(index_of(c));
        ++indeg[index_of(c)];
    }

    std::vector<std::vector<int>> result;
    std::vector<int> order;
    std::vector<char> placed(n, 0);
    order.reserve(n);
    // Depth-first, smallest available id first => lexicographic output.
    std::function<bool()> descend = [&]() -> bool {
        if (order.size() == n) {
            result.push_back(order);
            return result.size() < cap;
        }
        for (std::size_t i = 0; i < n; ++i) {
            if (placed[i] || indeg[i] != 0) continue;
            placed[i] = 1;
            order.push_back(ids[i]);
            for (std::size_t c : succ[i]) --indeg[c];
            const bool more = descend();
            for (std::size_t c : succ[i]) ++indeg[c];
            order.pop_back();
            placed[i] = 0;
            if (!more) return false;
        }
        return true;
    };
    descend();
    return result;
}

bool validate_sequence(const LayerDag& dag, const std::vector<int>& seq) {
    if (seq.size() != dag.nodes.size()) return false;
    std::map<int, std::size_t> at;
    for (std::size_t i = 0; i < seq.size(); ++i) {
        if (!at.emplace(seq[i], i).second) return false;
    }
    for (const auto& n : dag.nodes) {
        if (!at.count(n.id)) return false;
    }
    return std::all_of(dag.edges.begin(), dag.edges.end(),
                       [&](const std::pair<int, int>& e) { return at.at(e.first) < at.at(e.second); });
}

}  // namespace weft
