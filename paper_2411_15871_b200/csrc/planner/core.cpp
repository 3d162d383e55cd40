// L0 vocabulary: class/lane/pass names, default lanes, FNV-1a.
// Behaviour follows /root/reference/proj/src/presets.cpp:8-102.
#include "weft/core.hpp"

#include <array>

namespace weft {
namespace {

struct ClassInfo {
    std::string_view name;
    Lane lane;
};

// Indexed by static_cast<int>(OperatorClass).
constexpr std::array<ClassInfo, 13> kClasses{{
    {"GEMM", Lane::compute},
    {"FlashAttention", Lane::compute},
    {"FlashAttentionBwd", Lane::compute},
    {"GroupGEMM", Lane::compute},
    {"FusedBDA", Lane::compute},
    {"LayerNorm", Lane::compute},
    {"Router", Lane::compute},
    {"Permute", Lane::compute},
    {"WeightGrad", Lane::compute},
    {"AllGather", Lane::local_comm},
    {"ReduceScatter", Lane::local_comm},
    {"AllToAll", Lane::cross_comm},
    {"SendRecv", Lane::cross_comm},
}};

constexpr std::array<std::string_view, 3> kLanes{"compute", "local_comm", "cross_comm"};

}  // namespace

Lane default_lane(OperatorClass cls) {
    const auto i = static_cast<std::size_t>(cls);
    return i < kClasses.size() ? kClasses[i].lane : Lane::compute;
}

bool is_comm_class(OperatorClass cls) { return default_lane(cls) != Lane::compute; }

std::string_view to_string(OperatorClass cls) {
    const auto i = static_cast<std::size_t>(cls);
    return i < kClasses.size() ? kClasses[i].name : std::string_view("?");
}

OperatorClass parse_operator_class(std::string_view name) {
    for (std::size_t i = 0; i < kClasses.size(); ++i) {
        if (kClasses[i].name == name) return static_cast<OperatorClass>(i);
    }
    throw ConfigError("unknown operator class: " + std::string(name));
}

std::string_view to_string(Lane lane) {
    const auto i = static_cast<std::size_t>(lane);
    return i < kLanes.size() ? kLanes[i] : std::string_view("?");
}

Lane parse_lane(std::string_view name) {
    for (std::size_t i = 0; i < kLanes.size(); ++i) {
        if (kLanes[i] == name) return static_cast<Lane>(i);
    }
    throw ConfigError("unknown lane: " + std::string(name));
}

std::string_view to_string(Pass pass) {
    return pass == Pass::forward ? std::string_view("forward") : std::string_view("backward");
}

Pass parse_pass(std::string_view name) {
    if (name == "forward") return Pass::forward;
    if (name == "backward") return Pass::backward;
    throw ConfigError("unknown pass: " + std::string(name));
}

std::uint64_t fnv1a64(std::string_view data) {
    constexpr std::uint64_t kOffset = 14695981039346656037ull;
    constexpr std::uint64_t kPrime = 1099511628211ull;
    std::uint64_t h = kOffset;
    for (const char ch : data) {
        h = (h ^ static_cast<std::uint8_t>(ch)) * kPrime;
    }
    return h;
}

std::string hex64(std::uint64_t value) {
    constexpr char kHex[] = "0123456789abcdef";
    std::string s(16, '0');
    for (std::size_t k = 0; k < 16; ++k) {
        s[15 - k] = kHex[(value >> (4 * k)) & 0xfu];
    }
    return s;
}

}  // namespace weft
