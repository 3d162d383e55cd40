// Analytic collective volumes per iteration (drop-in for reference
// proj/src/comm_volume.cpp:6-67). Per-node wire bytes follow node_cost
// (op_model.cpp:290-301): TP/SP AG or RS moves tokens*h*2*(tp-1)/tp per GPU,
// 4 of each per layer pass pair; CP exchanges K and V around the ring; EP
// dispatch / combine move tokens*topk*h*2*(ep-1)/ep, twice each way; the DP
// gradient all-reduce moves 2*(dp-1)/dp of this GPU's bf16 gradients once.
#include "weft/comm_volume.hpp"

namespace weft {

double cross_time_ratio(double local_us, double cross_us) {
    const double sum = local_us + cross_us;
    return sum > 0.0 ? cross_us / sum : 0.0;
}

namespace {

struct Accumulator {
    const ClusterSpec& cl;
    CommVolume v;
    // bytes per GPU of one collective family spanning `extent` ranks
    void add(double bytes, int extent) {
        if (!(bytes > 0.0)) return;
        const bool in_node = extent <= cl.per_node;
        const double gbs = (in_node ? cl.local_bw_gbs : cl.cross_bw_gbs) * cl.bw_efficiency;
        const double us = bytes / (gbs * 1e3);
        auto& b = in_node ? v.local_bytes : v.cross_bytes;
        auto& t = in_node ? v.local_us : v.cross_us;
        b += static_cast<std::int64_t>(bytes);
        t += us;
    }
};

}  // namespace

CommVolume comm_volume_estimate(const ModelSpec& model, const ClusterSpec& cluster,
                                const ParallelismSpec& par, std::int64_t tokens_per_microbatch,
                                int microbatches) {
    model.validate();
    cluster.validate();
    par.validate(cluster);
    if (tokens_per_microbatch <= 0 || microbatches <= 0)
        throw ConfigError("comm_volume_estimate: tokens and microbatches must be positive");
    constexpr double kBytes = 2.0;  // bf16 on the wire
    const double tok = static_cast<double>(tokens_per_microbatch) / par.cp;
    const double hid = model.hidden;
    const double passes = static_cast<double>(model.layers) * microbatches;  // layer x micro-batch
    Accumulator acc{cluster, {}};
    if (par.tp > 1) {  // ag0 rs0 ag1 rs1 and their four backward counterparts
        const double per_op = tok * hid * kBytes * (par.tp - 1.0) / par.tp;
        acc.add(8.0 * per_op * passes, par.tp);
    }
    if (par.cp > 1) {  // K and V (h/tp columns each) to every other CP rank, fwd and bwd
        const double per_pass = 2.0 * tok * (hid / par.tp) * kBytes * (par.cp - 1.0);
        acc.add(2.0 * per_pass * passes, par.tp * par.cp);
    }
    if (par.ep > 1 && model.is_moe()) {  // a2a dispatch + combine, fwd and bwd
        const double per_op = tok * model.topk.value_or(1) * hid * kBytes * (par.ep - 1.0) / par.ep;
        acc.add(4.0 * per_op * passes, par.tp * par.cp * par.ep);
    }
    if (par.dp > 1) {  // ring all-reduce of this GPU's bf16 gradients, once
        const double grad_bytes =
            static_cast<double>(params_per_layer(model)) / par.tp * model.layers / par.pp * kBytes;
        acc.add(2.0 * grad_bytes * (par.dp - 1.0) / par.dp, par.tp * par.cp * par.dp);
    }
    acc.v.cross_time_ratio = cross_time_ratio(acc.v.local_us, acc.v.cross_us);
    return acc.v;
}

}  // namespace weft
