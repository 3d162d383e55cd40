// extern "C" JSON face of the planner (include/weft_capi.h).
//
// Compiled twice from this one source:
//   * into libweft_b200.so against our planner (namespace weft), symbols weft_*;
//   * by oracle/Makefile against the reference sources under /root/reference
//     with -Dweft=weft_ref -DWEFT_CAPI_REF, symbols weft_ref_* (the oracle).
// Both builds therefore answer byte-identical requests through identical glue,
// and parity tests compare the planners, not the adapters.
//
// Request schema (all keys optional unless noted):
//   model:        {name, family, hidden*, intermediate*, layers*, seq_len*, experts, topk}
//                 or {"preset": "llama-8B"}
//   parallelism:  {dp, tp, pp, cp, ep, sp}
//   cluster:      {name, gpus*, per_node*, peak_tflops*, local_bw_gbs*, cross_bw_gbs*,
//                  mem_gb*, bw_efficiency} or {"preset": "h100_32"}
//   profile:      a profile document (parse_profile schema) or {"archetype": "..."}
//   caps:         {sequences, segments, candidates}; barrier_cost_us, parallel, threads
//   metadata:     {str: str} passed to plan_to_json
//   schedule:     {discipline, m, p, f_us, b_us, si_us}            (pipeline_json)
//   memory:       {act_bytes_per_layer, state_bytes_per_layer, capacity_bytes,
//                  slack_bytes, layers} or {"defaults": true}      (memory_json)
//   source, microbatches, intra_batch_tp_hidden_frac              (estimate_json)
//   scenario:     a scenario document (parse_scenario schema)      (compare_json)
//   tokens, microbatches                                          (comm_volume_json)
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "nlohmann/json.hpp"
#include "weft/estimate.hpp"
#include "weft/folding_pipeline.hpp"
#include "weft/memory_sim.hpp"
#include "weft/op_model.hpp"
#include "weft/overlap_profile.hpp"
#include "weft/pairing_search.hpp"
#include "weft/presets.hpp"
#include "weft/comm_volume.hpp"
#include "weft/report.hpp"

#ifdef WEFT_CAPI_REF
#define WEFT_API(name) weft_ref_##name
#else
#define WEFT_API(name) weft_##name
#endif

using nlohmann::json;

namespace {

thread_local std::string g_error;

weft::ModelSpec model_from(const json& j) {
    if (j.contains("preset")) return weft::model_preset(j.at("preset").get<std::string>());
    weft::ModelSpec m;
    m.name = j.value("name", std::string("custom"));
    m.family = weft::parse_model_family(j.value("family", std::string("llama")));
    m.hidden = j.at("hidden").get<int>();
    m.intermediate = j.at("intermediate").get<int>();
    m.layers = j.at("layers").get<int>();
    m.seq_len = j.at("seq_len").get<int>();
    if (j.contains("experts") && !j.at("experts").is_null()) m.experts = j.at("experts").get<int>();
    if (j.contains("topk") && !j.at("topk").is_null()) m.topk = j.at("topk").get<int>();
    return m;
}

weft::ParallelismSpec par_from(const json& j) {
    weft::ParallelismSpec p;
    p.dp = j.value("dp", 1);
    p.tp = j.value("tp", 1);
    p.pp = j.value("pp", 1);
    p.cp = j.value("cp", 1);
    p.ep = j.value("ep", 1);
    p.sp = j.value("sp", false);
    return p;
}

weft::ClusterSpec cluster_from(const json& j) {
    if (j.contains("preset")) return weft::cluster_preset(j.at("preset").get<std::string>());
    weft::ClusterSpec c;
    c.name = j.value("name", std::string("custom"));
    c.gpus = j.at("gpus").get<int>();
    c.per_node = j.at("per_node").get<int>();
    c.peak_tflops = j.at("peak_tflops").get<double>();
    c.local_bw_gbs = j.at("local_bw_gbs").get<double>();
    c.cross_bw_gbs = j.at("cross_bw_gbs").get<double>();
    c.mem_gb = j.at("mem_gb").get<double>();
    c.bw_efficiency = j.value("bw_efficiency", 0.5);
    return c;
}

weft::Profile profile_from(const json& req) {
    if (!req.contains("profile")) return {};
    const json& j = req.at("profile");
    if (j.contains("archetype")) {
        return weft::synth_profile(weft::parse_archetype(j.at("archetype").get<std::string>()));
    }
    return weft::parse_profile(j.dump());
}

json node_json(const weft::OpNode& n) {
    return {{"id", n.id},
            {"class", std::string(weft::to_string(n.cls))},
            {"lane", std::string(weft::to_string(n.lane))},
            {"pass", std::string(weft::to_string(n.pass))},
            {"name", n.name},
            {"duration_us", n.duration_us},
            {"flops", n.flops},
            {"bytes", n.bytes}};
}

json dag_json(const weft::LayerDag& d) {
    json nodes = json::array(), edges = json::array();
    for (const auto& n : d.nodes) nodes.push_back(node_json(n));
    for (const auto& e : d.edges) edges.push_back({e.first, e.second});
    return {{"nodes", nodes}, {"edges", edges}, {"pass", std::string(weft::to_string(d.pass))}};
}

weft::OpNode node_from(const json& j) {
    weft::OpNode n;
    n.id = j.value("id", 0);
    n.cls = weft::parse_operator_class(j.at("class").get<std::string>());
    n.lane = j.contains("lane") ? weft::parse_lane(j.at("lane").get<std::string>())
                                : weft::default_lane(n.cls);
    n.pass = weft::parse_pass(j.value("pass", std::string("forward")));
    n.name = j.value("name", std::string());
    n.duration_us = j.value("duration_us", 0.0);
    n.flops = j.value("flops", 0.0);
    n.bytes = j.value("bytes", static_cast<std::int64_t>(0));
    return n;
}

weft::LayerDag dag_from(const json& j) {
    weft::LayerDag d;
    for (const auto& jn : j.at("nodes")) {
        if (jn.is_number_integer()) {
            weft::OpNode n;
            n.id = jn.get<int>();
            n.duration_us = 1.0;
            d.nodes.push_back(n);
        } else {
            d.nodes.push_back(node_from(jn));
        }
    }
    for (const auto& e : j.at("edges")) d.edges.emplace_back(e.at(0).get<int>(), e.at(1).get<int>());
    return d;
}

std::pair<weft::LayerDag, weft::LayerDag> dags_for(const json& req, const weft::Profile& prof) {
    const auto model = model_from(req.at("model"));
    const auto par = par_from(req.value("parallelism", json::object()));
    const auto cluster = cluster_from(req.at("cluster"));
    const bool use_solo = req.value("use_profile_solo", true);
    return weft::build_layer_dag(model, par, cluster, use_solo ? &prof.solo : nullptr);
}

json plan_json(const weft::PairingPlan& p) {
    json steps = json::array();
    for (const auto& s : p.steps) {
        steps.push_back({{"fwd_seg", s.fwd_seg ? json(*s.fwd_seg) : json(nullptr)},
                         {"bwd_seg", s.bwd_seg ? json(*s.bwd_seg) : json(nullptr)}});
    }
    return {{"steps", steps}, {"total_us", p.total_us}};
}

template <class Fn>
int guarded(const char* request, char** out, Fn&& fn) {
    if (out) *out = nullptr;
    try {
        const json req = json::parse(request ? request : "{}");
        const std::string text = fn(req).dump();
        char* buf = static_cast<char*>(std::malloc(text.size() + 1));
        if (!buf) throw std::bad_alloc();
        std::memcpy(buf, text.c_str(), text.size() + 1);
        *out = buf;
        return 0;
    } catch (const weft::ConfigError& e) {
        g_error = e.what();
        return 2;
    } catch (const weft::InfeasibleError& e) {
        g_error = e.what();
        return 3;
    } catch (const weft::MissingProfileEntry& e) {
        g_error = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_error = e.what();
        return 1;
    }
}

}  // namespace

extern "C" {

int WEFT_API(build_dag_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const auto prof = profile_from(req);
        const auto [fwd, bwd] = dags_for(req, prof);
        return json{{"fwd", dag_json(fwd)}, {"bwd", dag_json(bwd)}};
    });
}

int WEFT_API(topo_orders_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        weft::LayerDag dag;
        if (req.contains("dag")) {
            dag = dag_from(req.at("dag"));
        } else {
            const auto prof = profile_from(req);
            const auto both = dags_for(req, prof);
            dag = req.value("pass", std::string("forward")) == "backward" ? both.second : both.first;
        }
        const auto cap = req.value("cap", static_cast<std::size_t>(16));
        const auto orders = weft::enumerate_topological_orders(dag, cap);
        json valid = json::array();
        for (const auto& o : orders) valid.push_back(weft::validate_sequence(dag, o));
        return json{{"orders", orders}, {"valid", valid}};
    });
}

int WEFT_API(segment_cost_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const auto prof = profile_from(req);
        std::vector<weft::OpNode> a, b;
        for (const auto& j : req.at("a")) a.push_back(node_from(j));
        for (const auto& j : req.at("b")) b.push_back(node_from(j));
        const auto c = weft::segment_pair_cost(a, b, prof.overlap, prof.solo);
        return json{{"p_us", c.p_us}, {"lane_busy_us", c.lane_busy_us}};
    });
}

int WEFT_API(dp_align_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const int nf = req.at("n_f").get<int>(), nb = req.at("n_b").get<int>();
        const auto cost = req.at("cost").get<std::vector<std::vector<double>>>();
        const double barrier = req.value("barrier_cost_us", 0.0);
        weft::PairCostFn fn = [&](int i, int j) { return cost.at(i).at(j); };
        json r = {{"dp", plan_json(weft::dp_align(nf, nb, fn, barrier))}};
        if (req.value("brute_force", false)) {
            const auto bf = weft::brute_force_align(nf, nb, fn, barrier);
            r["brute_force"] = plan_json(bf.plan);
            r["alignments_enumerated"] = bf.alignments_enumerated;
        }
        return r;
    });
}

int WEFT_API(search_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const auto prof = profile_from(req);
        const auto [fwd, bwd] = dags_for(req, prof);
        weft::SearchOptions opt;
        if (req.contains("caps")) {
            const json& c = req.at("caps");
            opt.caps.sequences = c.value("sequences", opt.caps.sequences);
            opt.caps.segments = c.value("segments", opt.caps.segments);
            opt.caps.candidates = c.value("candidates", opt.caps.candidates);
        }
        opt.barrier_cost_us = req.value("barrier_cost_us", 0.0);
        opt.parallel = req.value("parallel", false);
        opt.threads = req.value("threads", 0);
        std::map<std::string, std::string> meta;
        if (req.contains("metadata")) meta = req.at("metadata").get<std::map<std::string, std::string>>();
        const int repeat = std::max(1, req.value("repeat", 1));
        weft::BestPlan best;
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < repeat; ++r) best = weft::search_si_plan(fwd, bwd, prof.overlap, prof.solo, opt);
        const auto t1 = std::chrono::steady_clock::now();
        const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count() / repeat;
        return json{{"plan_json", weft::plan_to_json(best, meta)},
                    {"candidates_evaluated", best.candidates_evaluated},
                    {"total_us", best.total_us},
                    {"hidden_comm_frac", best.hidden_comm_frac},
                    {"search_ms", ms},
                    {"fwd", dag_json(fwd)},
                    {"bwd", dag_json(bwd)}};
    });
}

int WEFT_API(profile_roundtrip_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const auto prof = profile_from(req);
        return json{{"profile_json", weft::profile_to_json(prof)}};
    });
}

const char* WEFT_API(last_error)(void) { return g_error.c_str(); }

void WEFT_API(free)(char* p) { std::free(p); }

}  // extern "C"

extern "C" int WEFT_API(templates_json)(const char* request, char** out) {
    return guarded(request, out, [](const json&) {
        return json{{"builtin_template_json", weft::builtin_template_json()}};
    });
}

namespace {

weft::PipelineSchedule schedule_from(const json& j) {
    const auto disc = weft::parse_discipline(j.value("discipline", std::string("w_shape")));
    const int m = j.at("m").get<int>(), p = j.at("p").get<int>();
    weft::BlockDurations d;
    d.f_us = j.value("f_us", d.f_us);
    d.b_us = j.value("b_us", d.b_us);
    d.si_us = j.value("si_us", d.si_us);
    switch (disc) {
        case weft::Discipline::w_shape: return weft::schedule_w_pipeline(m, p, d);
        case weft::Discipline::one_f_one_b: return weft::schedule_1f1b(m, p, d);
        case weft::Discipline::bidirectional: return weft::schedule_bidirectional(m, p, d);
    }
    throw weft::ConfigError("unknown discipline");
}

weft::MemoryConfig memory_from(const json& req) {
    const json& j = req.at("memory");
    weft::MemoryConfig c;
    if (j.value("defaults", false)) {
        const auto model = model_from(req.at("model"));
        const auto par = par_from(req.value("parallelism", json::object()));
        c.act_bytes_per_layer = weft::default_act_bytes_per_layer(model, par);
        c.state_bytes_per_layer = weft::default_state_bytes_per_layer(model, par);
        c.layers = model.layers;
    }
    c.act_bytes_per_layer = j.value("act_bytes_per_layer", c.act_bytes_per_layer);
    c.state_bytes_per_layer = j.value("state_bytes_per_layer", c.state_bytes_per_layer);
    c.capacity_bytes = j.value("capacity_bytes", c.capacity_bytes);
    c.slack_bytes = j.value("slack_bytes", c.slack_bytes);
    c.layers = j.value("layers", c.layers);
    return c;
}

}  // namespace

// fold_layers + schedule_* + analyses (reference folding_pipeline.hpp:23-103)
extern "C" int WEFT_API(pipeline_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const auto s = schedule_from(req.at("schedule"));
        json r = {{"trace_json", weft::schedule_to_trace_json(s)},
                  {"csv", weft::schedule_to_csv(s)},
                  {"makespan_us", s.makespan_us()},
                  {"bubble_ratio", weft::bubble_ratio(s)},
                  {"violations", weft::validate_schedule(s)},
                  {"pp_transfers", weft::pp_comm_volume(s, 1).transfers}};
        if (req.contains("fold_layers")) {
            const auto lay = weft::fold_layers(req.at("fold_layers").get<int>(), s.p);
            json g = json::array();
            for (const auto& x : lay.gpus) g.push_back({x.front_lo, x.front_hi, x.back_lo, x.back_hi});
            r["fold"] = g;
        }
        return r;
    });
}

// simulate_memory / max_model_size (reference memory_sim.hpp:47-79)
extern "C" int WEFT_API(memory_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const auto cfg = memory_from(req);
        json r = json::object();
        if (req.contains("schedule")) {
            const auto tl = weft::simulate_memory(schedule_from(req.at("schedule")), cfg);
            r["peaks_json"] = weft::peaks_to_json(tl, cfg);
            r["timeline_csv"] = weft::timeline_to_csv(tl);
        }
        if (req.contains("max_model")) {
            const json& mm = req.at("max_model");
            const auto res = weft::max_model_size(
                model_from(req.at("model")), par_from(req.value("parallelism", json::object())), cfg,
                weft::parse_discipline(mm.value("discipline", std::string("w_shape"))), mm.value("m", 8));
            r["max_layers"] = res.layers;
            r["max_params"] = res.param_count;
        }
        r["act_bytes_per_layer"] = cfg.act_bytes_per_layer;
        r["state_bytes_per_layer"] = cfg.state_bytes_per_layer;
        return r;
    });
}

// estimate_iteration_time (reference estimate.hpp:45-50)
extern "C" int WEFT_API(estimate_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const auto prof = profile_from(req);
        weft::EstimateOptions opt;
        opt.microbatches = req.value("microbatches", opt.microbatches);
        opt.intra_batch_tp_hidden_frac = req.value("intra_batch_tp_hidden_frac", opt.intra_batch_tp_hidden_frac);
        if (req.contains("caps")) {
            const json& c = req.at("caps");
            opt.search.caps.sequences = c.value("sequences", opt.search.caps.sequences);
            opt.search.caps.segments = c.value("segments", opt.search.caps.segments);
            opt.search.caps.candidates = c.value("candidates", opt.search.caps.candidates);
        }
        const auto r = weft::estimate_iteration_time(
            model_from(req.at("model")), cluster_from(req.at("cluster")),
            par_from(req.value("parallelism", json::object())),
            weft::parse_plan_source(req.value("source", std::string("dhelix"))), prof, opt);
        return json{{"makespan_us", r.makespan_us},   {"tflops_per_gpu", r.tflops_per_gpu},
                    {"mfu", r.mfu},                   {"hidden_comm_frac", r.hidden_comm_frac},
                    {"layer_fwd_us", r.layer_fwd_us}, {"layer_bwd_us", r.layer_bwd_us},
                    {"layer_pair_us", r.layer_pair_us}};
    });
}

// compare_report on a scenario document (reference report.hpp:56-63)
extern "C" int WEFT_API(compare_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const weft::Scenario sc = weft::parse_scenario(req.at("scenario").dump());
        const weft::CompareReport rep = weft::compare_report(sc);
        return json{{"report_json", weft::report_to_json(rep)},
                    {"report_csv", weft::report_to_csv(rep)},
                    {"config_hash", rep.config_hash},
                    {"canonical_json", sc.canonical_json()}};
    });
}

// comm_volume_estimate (reference comm_volume.hpp:26-29)
extern "C" int WEFT_API(comm_volume_json)(const char* request, char** out) {
    return guarded(request, out, [](const json& req) {
        const auto v = weft::comm_volume_estimate(
            model_from(req.at("model")), cluster_from(req.at("cluster")),
            par_from(req.value("parallelism", json::object())), req.at("tokens").get<std::int64_t>(),
            req.value("microbatches", 1));
        return json{{"local_bytes", v.local_bytes}, {"cross_bytes", v.cross_bytes}, {"local_us", v.local_us},
                    {"cross_us", v.cross_us}, {"cross_time_ratio", v.cross_time_ratio}};
    });
}
