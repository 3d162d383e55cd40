// L1 specs: validation, parameter count and the preset catalogs.
// Behaviour follows /root/reference/proj/src/presets.cpp:104-270 (messages,
// validation order and catalog contents are part of the contract; the
// reference tests look presets up by name).
#include "weft/presets.hpp"

#include <algorithm>

namespace weft {

std::string_view to_string(ModelFamily family) {
    switch (family) {
        case ModelFamily::llama: return "llama";
        case ModelFamily::gpt: return "gpt";
        case ModelFamily::phi_moe: return "phi_moe";
    }
    return "?";
}

ModelFamily parse_model_family(std::string_view name) {
    static constexpr std::pair<std::string_view, ModelFamily> kMap[] = {
        {"llama", ModelFamily::llama}, {"gpt", ModelFamily::gpt}, {"phi_moe", ModelFamily::phi_moe}};
    for (const auto& [n, f] : kMap) {
        if (n == name) return f;
    }
    throw ConfigError("unknown model family: " + std::string(name));
}

void ModelSpec::validate() const {
    const bool dims_ok = hidden > 0 && intermediate > 0 && layers > 0 && seq_len > 0;
    if (!dims_ok) throw ConfigError("model '" + name + "': dimensions must be positive");
    const bool moe_family = family == ModelFamily::phi_moe;
    const int e = experts.value_or(0);
    if (moe_family && e < 2) throw ConfigError("model '" + name + "': phi_moe needs experts >= 2");
    if (!moe_family && experts && e > 1) {
        throw ConfigError("model '" + name + "': experts set on a dense family");
    }
}

void ClusterSpec::validate() const {
    const bool positive = gpus > 0 && per_node > 0 && peak_tflops > 0.0 && local_bw_gbs > 0.0 &&
                          cross_bw_gbs > 0.0 && mem_gb > 0.0;
    if (!positive) throw ConfigError("cluster '" + name + "': fields must be positive");
    if (gpus % per_node) throw ConfigError("cluster '" + name + "': gpus not divisible by per_node");
    if (!(bw_efficiency > 0.0 && bw_efficiency <= 1.0)) {
        throw ConfigError("cluster '" + name + "': bw_efficiency must be in (0, 1]");
    }
}

void ParallelismSpec::validate() const {
    if (std::min({dp, tp, pp, cp, ep}) < 1) {
        throw ConfigError("parallelism group sizes must be >= 1");
    }
    if (dp % ep) throw ConfigError("ep must divide dp (EP group is a subset of the DP group)");
    if (sp && tp < 2) throw ConfigError("sp requires tp > 1");
}

void ParallelismSpec::validate(const ClusterSpec& cluster) const {
    validate();
    const int n = total_gpus();
    if (n != cluster.gpus) {
        throw ConfigError("dp*tp*pp*cp = " + std::to_string(n) + " does not match cluster gpus = " +
                          std::to_string(cluster.gpus));
    }
}

std::int64_t params_per_layer(const ModelSpec& m) {
    const std::int64_t h = m.hidden, f = m.intermediate;
    const std::int64_t base = 4 * h * h + 2 * h;  // qkv + out-proj + two norm vectors
    if (m.family == ModelFamily::llama) return base + 3 * h * f;
    if (m.family == ModelFamily::gpt) return base + 2 * h * f;
    if (m.family == ModelFamily::phi_moe) {
        const std::int64_t e = m.experts.value_or(1);
        return base + e * (3 * h * f + h);
    }
    return 0;
}

namespace {

struct ModelRow {
    const char* name;
    ModelFamily family;
    int hidden, intermediate, layers, seq;
    int experts, topk;  // 0 = unset
};

constexpr ModelRow kModels[] = {
    {"llama-8B", ModelFamily::llama, 4096, 14336, 32, 8192, 0, 0},
    {"llama-25B", ModelFamily::llama, 8192, 28672, 28, 8192, 0, 0},
    {"llama-39B", ModelFamily::llama, 16384, 53248, 12, 8192, 0, 0},
    {"llama-66B", ModelFamily::llama, 8192, 28672, 76, 16384, 0, 0},
    {"gpt-6.7B", ModelFamily::gpt, 4096, 16384, 32, 8192, 0, 0},
    {"gpt-18B", ModelFamily::gpt, 6144, 24576, 40, 8192, 0, 0},
    {"gpt-30B", ModelFamily::gpt, 12288, 49152, 16, 8192, 0, 0},
    {"phi-16B", ModelFamily::phi_moe, 4096, 6400, 12, 3072, 16, 2},
    {"phi-31B", ModelFamily::phi_moe, 4096, 6400, 24, 3072, 16, 2},
    {"phi-42B", ModelFamily::phi_moe, 4096, 6400, 32, 3072, 16, 2},
};

struct ClusterRow {
    const char* name;
    int gpus, per_node;
    double peak, local_bw, cross_bw, mem;
};

constexpr ClusterRow kClusters[] = {
    {"a40_64", 64, 8, 149.7, 32.0, 12.5, 48.0},
    {"a800_64", 64, 8, 312.0, 400.0, 100.0, 80.0},
    {"a100_8", 8, 8, 312.0, 600.0, 12.5, 80.0},
    {"h100_32", 32, 8, 989.0, 900.0, 400.0, 80.0},
};

ModelSpec to_spec(const ModelRow& r) {
    ModelSpec m;
    m.name = r.name;
    m.family = r.family;
    m.hidden = r.hidden;
    m.intermediate = r.intermediate;
    m.layers = r.layers;
    m.seq_len = r.seq;
    if (r.experts) m.experts = r.experts;
    if (r.topk) m.topk = r.topk;
    return m;
}

ClusterSpec to_spec(const ClusterRow& r) {
    ClusterSpec c;
    c.name = r.name;
    c.gpus = r.gpus;
    c.per_node = r.per_node;
    c.peak_tflops = r.peak;
    c.local_bw_gbs = r.local_bw;
    c.cross_bw_gbs = r.cross_bw;
    c.mem_gb = r.mem;
    return c;
}

}  // namespace

ModelSpec model_preset(const std::string& name) {
    for (const auto& r : kModels) {
        if (name == r.name) return to_spec(r);
    }
    throw ConfigError("unknown model preset: " + name);
}

ClusterSpec cluster_preset(const std::string& name) {
    for (const auto& r : kClusters) {
        if (name == r.name) return to_spec(r);
    }
    throw ConfigError("unknown cluster preset: " + name);
}

std::vector<std::string> model_preset_names() {
    std::vector<std::string> out;
    for (const auto& r : kModels) out.emplace_back(r.name);
    return out;
}

std::vector<std::string> cluster_preset_names() {
    std::vector<std::string> out;
    for (const auto& r : kClusters) out.emplace_back(r.name);
    return out;
}

}  // namespace weft
