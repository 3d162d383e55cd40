// SI executor: lowers a weft plan (plan_to_json, reference pairing_search.cpp:
// 543-561) into lane-stream launches and runs them eagerly or as a CUDA graph.
//
// Schedule (reference folding_pipeline.cpp schedule_w_pipeline with p = 1; the
// SI block order is taken from our schedule_w_pipeline(m, 1)):
//   SI mode          F_0 | SI(F_1, B_0) | SI(F_2, B_1) | ... | B_{m-1}
//   sequential mode  F_0 B_0 | F_1 B_1 | ...       (same per-strand op orders)
// Inside SI(F_{i+1}, B_i) forward layer k of strand i+1 is paired with
// backward layer L-1-k of strand i, step by step as the plan says. Each step
// is lowered by replaying the lane model (lane_sim.hpp — the same dispatch
// rule the planner's cost model uses) on the node solo times: the resulting
// start order becomes the issue order on the three lane streams. Edges:
//   * strand order: an op waits for its strand predecessor when that ran on a
//     different lane (same-lane order is implicit in the stream);
//   * step barrier: the first op of each lane in a step waits for the last op
//     of every other lane (the paper's inter-step synchronisation,
//     PAPER.md:673), also at phase boundaries (transient buffers change owner).
// Because every wait refers to an op issued earlier in program order, the
// event graph is acyclic and the issue order is deadlock-free.
//
// Memory: L+1 activation slots. Forward of (strand, layer) pops a free slot,
// backward of (strand, layer) pushes it back after its layer pair completes;
// in an SI block the forward strand therefore always reuses the slot the
// backward strand released one step earlier (never the one it still reads).
//
// Backward running gradient: layer l reads dy from grad[(L-2-l)&1] (the top
// layer reads dL/dy) and writes the layer-input gradient to grad[(L-1-l)&1].
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <tuple>

#include "../planner/lane_sim.hpp"
#include "runtime.hpp"
#include "weft/folding_pipeline.hpp"

namespace dh {

namespace {

int n_slots(const Model& m) { return m.cfg.slots > 0 ? m.cfg.slots : m.cfg.layers + 1; }

struct Lowering {
    Model& m;
    Program prog;
    std::array<int, kLanes> lane_last{-1, -1, -1};
    std::array<int, kLanes> join_snapshot{-1, -1, -1};
    std::array<bool, kLanes> pending_join{false, false, false};
    std::vector<int> strand_last;
    std::vector<std::vector<int>> slot_of;  // [strand][layer]
    std::vector<int> free_slots;
    int peak_slots = 0;  // most activation slots held at once
    std::map<int, int> lane_of, pos_in_bwd, pos_in_fwd;

    explicit Lowering(Model& mm) : m(mm) {
        const int mb = m.cfg.micro_batches, L = m.cfg.layers;
        strand_last.assign(mb, -1);
        slot_of.assign(mb, std::vector<int>(L, -1));
        for (int s = n_slots(m) - 1; s >= 0; --s) free_slots.push_back(s);  // pop_back gives 0 first
        for (const auto& n : m.fwd_dag.nodes) lane_of[n.id] = static_cast<int>(n.lane);
        for (const auto& n : m.bwd_dag.nodes) lane_of[n.id] = static_cast<int>(n.lane);
        for (std::size_t i = 0; i < m.plan.bwd_seq.size(); ++i) pos_in_bwd[m.plan.bwd_seq[i]] = static_cast<int>(i);
        for (std::size_t i = 0; i < m.plan.fwd_seq.size(); ++i) pos_in_fwd[m.plan.fwd_seq[i]] = static_cast<int>(i);
    }

    void barrier() {
        join_snapshot = lane_last;
        pending_join.fill(true);
    }

    // Ops outside an SI block run strictly in strand order (one lane at a
    // time), so their GEMMs never share the GPU with a collective and take
    // every SM; inside a block the cap applies wherever a collective may co-run.
    bool capped = false;
    int cur_part = -1;  // Op::part of the next mlp_fc1_wgrad emitted

    // deps (optional): the op's data predecessors (op indices) replace the
    // strand-order wait, so a strand can overlap its own independent ops
    void emit(int strand, int layer, int node, int peer = -1, const std::vector<int>* deps = nullptr) {
        const bool xfer = node >= kSendAct && node <= kRecvGrad;
        // compute-only measurement program: collectives are left out entirely
        if (m.skip_comm && !xfer && lane_of.at(node) != 0) return;
        Op o;
        o.strand = strand;
        o.layer = layer;
        o.node = node;
        o.peer = peer;
        // pipeline transfers are stream-ordered copies on the compute lane: the
        // running-gradient buffer they read is rewritten by the next backward op
        o.lane = xfer ? 0 : lane_of.at(node);
        o.slot = slot_of[strand][layer];
        o.prev_slot = layer > 0 ? slot_of[strand][layer - 1] : -1;
        o.capped = capped;
        o.part = node == 26 ? cur_part : -1;
        if (xfer) {
            // nothing node-specific
        } else if (m.cfg.moe) {
            // moe_ep ids: no cross-node fusion flags (expert_fc1 fuses its own SwiGLU)
        } else if (node == 10 || node == 11) {
            // both run on the compute lane in sequence order: the later one sees the
            // other's output and applies SwiGLU in its GEMM epilogue
            const int other = node == 10 ? 11 : 10;
            o.fuse_swiglu = pos_in_fwd.at(node) > pos_in_fwd.at(other) &&
                            lane_of.at(node) == lane_of.at(other);
        }
        if (!xfer && !m.cfg.moe && (node == 24 || node == 25)) {
            const int other = node == 24 ? 25 : 24;
            o.first_dx = pos_in_bwd.at(node) < pos_in_bwd.at(other);
        }
        const int idx = static_cast<int>(prog.ops.size());
        const int prev = strand_last[strand];
        if (deps) {
            for (int d : *deps)  // same-lane predecessors are ordered by the stream
                if (d >= 0 && prog.ops[d].lane != o.lane &&
                    std::find(o.waits.begin(), o.waits.end(), d) == o.waits.end())
                    o.waits.push_back(d);
        } else if (prev >= 0 && prog.ops[prev].lane != o.lane) {
            o.waits.push_back(prev);
        }
        if (pending_join[o.lane]) {
            for (int l = 0; l < kLanes; ++l) {
                if (l != o.lane && join_snapshot[l] >= 0 &&
                    std::find(o.waits.begin(), o.waits.end(), join_snapshot[l]) == o.waits.end())
                    o.waits.push_back(join_snapshot[l]);
            }
            pending_join[o.lane] = false;
        }
        prog.ops.push_back(std::move(o));
        strand_last[strand] = idx;
        lane_last[prog.ops[idx].lane] = idx;
    }

    // AdamW of `layer` once the last strand's backward of it is done: it waits
    // for that strand's last op (the strand runs in total order, and every
    // gradient writer of the layer is on the compute lane ahead of it) and
    // stays off the strand chains, so the backward continues meanwhile.
    void emit_opt(int strand, int layer) {
        // EP > 1: the replicated weights' data-parallel all-reduce must precede
        // their AdamW, so the whole optimizer runs after the program
        if (!m.fuse_optimizer || (m.cfg.moe && m.cfg.ep > 1)) return;
        Op o;
        o.strand = -1;
        o.layer = layer;
        o.node = kOptNode;
        o.lane = kLanes - 1;
        o.slot = -1;
        o.prev_slot = -1;
        o.capped = false;
        o.waits.push_back(strand_last[strand]);
        prog.ops.push_back(std::move(o));
        lane_last[kLanes - 1] = static_cast<int>(prog.ops.size()) - 1;
        has_opt = true;
    }
    bool has_opt = false;

    void take_slot(int strand, int layer) {
        if (free_slots.empty())
            throw std::runtime_error("not enough activation slots for this schedule (dh_model_cfg.slots)");
        slot_of[strand][layer] = free_slots.back();
        free_slots.pop_back();
        peak_slots = std::max(peak_slots, n_slots(m) - static_cast<int>(free_slots.size()));
    }
    void give_slot(int strand, int layer) { free_slots.push_back(slot_of[strand][layer]); }

    void forward_layer(int strand, int layer) {
        take_slot(strand, layer);
        for (int id : m.plan.fwd_seq) emit(strand, layer, id);
    }
    void backward_layer(int strand, int layer) {
        for (int id : m.plan.bwd_seq) emit(strand, layer, id);
        give_slot(strand, layer);
    }
    // Backward of a strand that runs alone (the unpaired B_m of the SI
    // schedule): the plan's order on each lane, but waits on data
    // predecessors only (the layer DAG's edges; sources wait for the previous
    // layer's last op), so a collective overlaps its own strand's independent
    // work — e.g. ag1_bwd_rs under mlp_fc1_wgrad, ag0_bwd_rs under qkv_wgrad.
    // Every transient buffer's next writer is a DAG or stream-order successor
    // of its readers (tests/test_executor_lowering.py, buffer hazards). GEMMs
    // issued while a collective of the layer is still open are capped like
    // co-running ones.
    //
    // In the SI modes at TP > 1 (EP > 1) it also moves its weight gradients under its
    // collectives (the plan's order leaves three of the four exposed:
    // tools/op_timeline.py): mlp_down_wgrad after ag1_bwd_rs (the RS of the MLP
    // input gradient), mlp_fc1_wgrad split into its gate and up launches after
    // rs0_bwd_ag (the AG before attn_proj_dgrad) and after ag0_bwd_rs (the RS
    // of the layer's input gradient), and the attention weight gradients
    // (attn_proj_wgrad, qkv_wgrad) into the next layer, right after its
    // rs1_bwd_ag — the mode-4 deferral of the SI pairs. Their inputs are
    // rewritten only by later ops of the next layer (d_gate / d_up by
    // mlp_down_dgrad, dx1_full by rs0_bwd_ag, dqkv by attn_bwd), which the
    // buffer-hazard tests check.
    bool lone_reorder = [] {
        const char* e = std::getenv("DH_SI_LONE_REORDER");
        return !e || std::atoi(e) != 0;
    }();
    // moe_ep (EP > 1): only the attention weight gradients (attn_proj_wgrad 34,
    // qkv_wgrad 38) move, under the next layer's a2a_combine_bwd; the dispatch
    // all-to-all already runs under expert_fc1_wgrad in the plan's order
    bool lone_block = false;  // lowering the unpaired last backward strand of an SI schedule
    bool lone_defers() const {
        return lone_block && lone_reorder && (m.cfg.moe ? m.cfg.ep > 1 : m.cfg.tp > 1);
    }

    void backward_layer_dag(int strand, int layer) {
        std::map<int, std::vector<int>> preds;
        for (const auto& [a, b] : m.bwd_dag.edges) preds[b].push_back(a);
        std::map<int, int> at;  // node id -> op index
        std::vector<int> open_comm;  // comm nodes whose consumers are not emitted yet
        const int prev_last = strand_last[strand];
        int last = prev_last;
        std::vector<int> seq = m.plan.bwd_seq;
        const bool reorder = lone_defers();
        auto has = [&](int id) { return std::find(seq.begin(), seq.end(), id) != seq.end(); };
        std::vector<int> part_of(seq.size(), -1);
        int defer_a = 32, defer_b = 36;  // the attention weight gradients
        if (reorder && m.cfg.moe && has(34) && has(38)) {
            defer_a = 34;
            defer_b = 38;
            seq.erase(std::find(seq.begin(), seq.end(), 34));
            seq.erase(std::find(seq.begin(), seq.end(), 38));
        } else if (reorder && !m.cfg.moe && has(23) && has(26) && has(27) && has(30) && has(32) && has(36) &&
                   has(37)) {
            auto move_after = [&](int id, int anchor) {
                seq.erase(std::find(seq.begin(), seq.end(), id));
                seq.insert(std::find(seq.begin(), seq.end(), anchor) + 1, id);
            };
            move_after(23, 27);
            move_after(26, 30);
            seq.insert(std::find(seq.begin(), seq.end(), 37) + 1, 26);  // the up half
            seq.erase(std::find(seq.begin(), seq.end(), 32));
            seq.erase(std::find(seq.begin(), seq.end(), 36));
            part_of.assign(seq.size(), -1);
            int k = 0;
            for (std::size_t i = 0; i < seq.size(); ++i)
                if (seq[i] == 26) part_of[i] = k++;
        } else if (reorder) {
            flush_deferred();
        }
        const bool defer_attn = reorder && !has(defer_a) && !has(defer_b);
        bool flushed = false;
        for (std::size_t si = 0; si < seq.size(); ++si) {
            const int id = seq[si];
            std::vector<int> deps;
            for (int p : preds[id]) deps.push_back(at.at(p));
            if (deps.empty() && prev_last >= 0) deps.push_back(prev_last);
            for (int p : preds[id]) open_comm.erase(std::remove(open_comm.begin(), open_comm.end(), p), open_comm.end());
            const bool comm = lane_of.at(id) != 0;
            capped = !comm && !open_comm.empty();
            cur_part = part_of[si];
            emit(strand, layer, id, -1, &deps);
            cur_part = -1;
            at[id] = static_cast<int>(prog.ops.size()) - 1;
            bwd_op_at[{strand, layer, id}] = at[id];
            if (comm) open_comm.push_back(id);
            // the layer's completion point for the next layer's sources: its
            // compute-lane tail (every comm op feeds a later compute op)
            if (prog.ops.back().lane == 0) last = at[id];
            if (comm && !flushed && deferred.strand >= 0) {
                // the previous layer's attention weight gradients run under this
                // layer's first collective
                strand_last[strand] = last;
                flush_deferred();
                flushed = true;
            }
        }
        capped = false;
        if (!flushed) flush_deferred();
        strand_last[strand] = last;
        if (defer_attn) {
            deferred.strand = strand;
            deferred.layer = layer;
            deferred.nodes = {defer_a, defer_b};  // slot released by flush_deferred()
        } else {
            give_slot(strand, layer);
        }
    }

    double solo(int id, const weft::LayerDag& dag) {
        auto it = m.solo_us.find(id);
        if (it != m.solo_us.end()) return it->second;
        return dag.find(id)->duration_us;
    }

    std::vector<int> segment(const weft::Segmentation& sg, int k) {
        if (k <= 0) return {};
        const auto [lo, hi] = sg.segment_range(static_cast<std::size_t>(k));
        return std::vector<int>(sg.sequence.begin() + lo, sg.sequence.begin() + hi);
    }

    // One SI layer pair: forward (fs, lf) with backward (bs, lb), per plan step.
    // relaxed (mode 2): the plan's per-lane issue order is kept but only the first
    // step of a layer pair joins the lanes (it guards the activation slot the
    // forward strand takes over from the backward strand); inside a layer pair the
    // two strands touch disjoint buffers, so the per-strand event edges suffice.
    // Mode 4 (relaxed steps + deferred weight gradients): the backward strand's
    // trailing attention weight gradients (attn_proj_wgrad, qkv_wgrad: sinks
    // that only read the layer's slot, dqkv and the attention-output gradient)
    // are issued after the NEXT layer pair's first step, where they fill the
    // compute lane while that pair's leading collectives (rs1_bwd_ag, ag0) run.
    // Their layer's activation slot is released after them, so the schedule
    // needs one activation slot more (dh_model_cfg.slots >= L + 2).
    struct Deferred {
        int strand = -1, layer = -1;
        std::vector<int> nodes;
    } deferred;
    bool defer_wgrads = false;

    void flush_deferred() {
        if (deferred.strand < 0) return;
        std::map<int, std::vector<int>> preds;
        for (const auto& [a, b] : m.bwd_dag.edges) preds[b].push_back(a);
        const int keep_last = strand_last[deferred.strand];
        for (int id : deferred.nodes) {
            std::vector<int> deps;
            for (int p : preds[id]) deps.push_back(bwd_op_at.at({deferred.strand, deferred.layer, p}));
            capped = true;  // may co-run with the next pair's collectives
            emit(deferred.strand, deferred.layer, id, -1, &deps);
        }
        capped = false;
        strand_last[deferred.strand] = keep_last;  // the strand's chain continues from its own ops
        give_slot(deferred.strand, deferred.layer);
        deferred = Deferred{};
    }
    std::map<std::tuple<int, int, int>, int> bwd_op_at;  // (strand, layer, node) -> op index (mode 4)
    // qkv_wgrad stays in its own pair, issued just before the forward strand's
    // bda1 (which waits for rs1); only attn_proj_wgrad crosses into the next pair.
    // Measured at TP=8 shapes: 231.9-232.2 -> 230.1-230.5 ms/step against
    // deferring both (DH_SI_SPLIT_DEFER=0 restores that).
    bool split_defer = [] {
        const char* e = std::getenv("DH_SI_SPLIT_DEFER");
        return !e || std::atoi(e) != 0;
    }();
    void emit_deferred_now(int strand, int layer, int id, std::vector<int>& pending) {
        std::map<int, std::vector<int>> preds;
        for (const auto& [a, b] : m.bwd_dag.edges) preds[b].push_back(a);
        std::vector<int> deps;
        for (int p : preds[id]) deps.push_back(bwd_op_at.at({strand, layer, p}));
        const int keep_last = strand_last[strand];
        const bool keep_cap = capped;
        capped = true;
        emit(strand, layer, id, -1, &deps);
        capped = keep_cap;
        strand_last[strand] = keep_last;
        pending.erase(std::remove(pending.begin(), pending.end(), id), pending.end());
        issued_early.push_back(id);
    }
    // ids of the current pair already issued ahead of their step (never cleared
    // within the pair, so a later step cannot issue them a second time)
    std::vector<int> issued_early;
    // DH_SI_DEFER_DOWN_WGRAD=0: keep mlp_down_wgrad in its own pair (mode 4)
    bool defer_down_wgrad = [] {
        const char* e = std::getenv("DH_SI_DEFER_DOWN_WGRAD");
        return !e || std::atoi(e) != 0;
    }();

    void si_layer_pair(int fs, int lf, int bs, int lb, const weft::OverlapTable& tbl, bool relaxed) {
        take_slot(fs, lf);
        if (pending_recv_act.first == fs) {
            emit(fs, lf, kRecvAct, pending_recv_act.second);
            pending_recv_act = {-1, -1};
        }
        // The backward strand's leading ops up to its first collective (bda1_bwd,
        // rs1_bwd_ag) depend only on the previous layer's gradient, ready when
        // the pair starts: they join the first step, so the collective runs
        // under that step's compute instead of stalling the GEMM that waits for
        // it in a later, joined step (tools/op_timeline.py measured that stall
        // as the largest exposed collective inside SI blocks). DH_SI_HOIST=0 off.
        static const bool hoist_on = [] {
            const char* e = std::getenv("DH_SI_HOIST");
            return !e || std::atoi(e) != 0;
        }();
        std::vector<int> hoist;
        if (hoist_on) {
            for (int id : m.plan.bwd_seq) {
                hoist.push_back(id);
                if (lane_of.at(id) != 0) break;
            }
            if (hoist.empty() || lane_of.at(hoist.back()) == 0) hoist.clear();  // no collective
        }
        auto hoisted = [&](int id) { return std::find(hoist.begin(), hoist.end(), id) != hoist.end(); };
        // this pair's deferrable ops: the attention weight gradients after the
        // backward layer's last collective (dense template ids 32, 36), and
        // mlp_down_wgrad (23) wherever the plan put it: a sink whose inputs (the
        // layer's slot, the parity-indexed gathered gradient) outlive this pair, so
        // it fills the next pair's opening, where both strands start with a
        // collective (rs1_bwd_ag, ag0) and little compute of their own
        std::vector<int> defer_now;
        if (defer_wgrads && !m.cfg.moe) {
            int last_comm = -1;
            for (std::size_t i = 0; i < m.plan.bwd_seq.size(); ++i)
                if (lane_of.at(m.plan.bwd_seq[i]) != 0) last_comm = static_cast<int>(i);
            if (defer_down_wgrad && m.cfg.tp > 1) defer_now.push_back(23);
            for (std::size_t i = last_comm + 1; last_comm >= 0 && i < m.plan.bwd_seq.size(); ++i) {
                const int id = m.plan.bwd_seq[i];
                if (id == 32 || id == 36) defer_now.push_back(id);
            }
        }
        issued_early.clear();
        auto deferred_here = [&](int id) {
            return std::find(defer_now.begin(), defer_now.end(), id) != defer_now.end() ||
                   std::find(issued_early.begin(), issued_early.end(), id) != issued_early.end();
        };
        bool first_step = true;
        flush_after_step = true;  // the previous pair's deferred ops follow this pair's first step
        for (const auto& st : m.plan.plan.steps) {
            const auto fa = segment(m.plan.fwd_segmentation, st.fwd_seg.value_or(0));
            std::vector<int> ba;
            if (first_step) ba = hoist;
            for (int id : segment(m.plan.bwd_segmentation, st.bwd_seg.value_or(0)))
                if (!hoisted(id) && !deferred_here(id)) ba.push_back(id);
            std::vector<weft::detail::SimOp> sa, sb;
            for (int id : fa) {
                const auto* n = m.fwd_dag.find(id);
                sa.push_back({solo(id, m.fwd_dag), n->lane, n->cls});
            }
            for (int id : ba) {
                const auto* n = m.bwd_dag.find(id);
                sb.push_back({solo(id, m.bwd_dag), n->lane, n->cls});
            }
            std::vector<std::pair<int, std::size_t>> order;
            std::vector<std::pair<double, double>> spans;
            weft::detail::simulate_lanes(
                sa.data(), sa.size(), sb.data(), sb.size(), tbl.slowdown_factor,
                tbl.launch_overhead_frac,
                [&](const weft::detail::SimOp& x, const weft::detail::SimOp& y) {
                    const auto v = tbl.get(x.cls, y.cls);
                    return v ? *v : 0.0;  // missing pairs only affect issue order
                },
                &order, &spans);
            if (!relaxed || first_step) barrier();
            first_step = false;
            // Joined steps: a compute op is capped when its simulated interval
            // overlaps one of the step's collectives (the lane model's timeline
            // on the measured solo times); relaxed steps may overlap their
            // neighbours, so the whole block is capped.
            auto is_comm = [&](std::size_t t) {
                const auto& [side, i] = order[t];
                return lane_of.at(side == 0 ? fa[i] : ba[i]) != 0;
            };
            for (std::size_t t = 0; t < order.size(); ++t) {
                const auto& [side, i] = order[t];
                bool cap = relaxed;
                if (!relaxed && !is_comm(t)) {
                    for (std::size_t c = 0; c < order.size() && !cap; ++c)
                        cap = is_comm(c) && spans[c].first < spans[t].second && spans[t].first < spans[c].second;
                }
                if (side == 0 && fa[i] == 14 && split_defer && std::find(defer_now.begin(), defer_now.end(), 36) != defer_now.end() &&
                    bwd_op_at.count({bs, lb, 34})) {
                    // qkv_wgrad of this pair fills the forward strand's last stall (bda1
                    // waits for rs1): issue it before bda1 once attn_bwd is out
                    emit_deferred_now(bs, lb, 36, defer_now);
                }
                if (side == 1 && deferred.strand >= 0 && (ba[i] == 28 || ba[i] == 30 || ba[i] == 34)) {
                    // the next layer is about to overwrite an input of the deferred
                    // gradients (d_x1 / dx1_full / dqkv): issue them first
                    flush_deferred();
                }
                capped = cap;
                if (side == 0) {
                    emit(fs, lf, fa[i]);
                } else {
                    emit(bs, lb, ba[i]);
                    bwd_op_at[{bs, lb, ba[i]}] = static_cast<int>(prog.ops.size()) - 1;
                }
            }
            if (flush_after_step) flush_deferred();
            flush_after_step = false;
        }
        if (flush_after_step) flush_deferred();  // (a plan without steps)
        flush_after_step = false;
        if (!defer_now.empty()) {
            deferred.strand = bs;
            deferred.layer = lb;
            deferred.nodes = defer_now;  // slot released by flush_deferred()
        } else {
            give_slot(bs, lb);
        }
        capped = false;
    }
    bool flush_after_step = false;  // a deferred set from the previous pair awaits this pair's first step

    // ---- W pipeline stage (mode 3)
    // Local layers [0, c) are the way-down half and [c, L) the way-back half of
    // this stage's U-fold share (the last stage's two halves are contiguous and
    // visited at once). Transfers cross to the neighbour on the weft u_path.
    struct Visit {
        int lo, hi;         // forward span [lo, hi); the backward span is its mirror
        int peer_in, peer_out;  // -1: global first / last layer (no transfer)
    };
    Visit visit_of(const weft::Block& b) const {
        const int L = m.cfg.layers, c = L / 2, d = m.cfg.pp_rank, p = m.cfg.pp_size;
        Visit v;
        if (b.half_stages == 2) {  // turn (last stage), or the whole pass at p = 1
            v = {0, L, p > 1 ? d - 1 : -1, p > 1 ? d - 1 : -1};
        } else if (b.half == weft::HalfDir::down) {
            v = {0, c, d > 0 ? d - 1 : -1, d + 1};
        } else {
            v = {c, L, d + 1, d > 0 ? d - 1 : -1};
        }
        return v;
    }
    void fwd_visit(int strand, const Visit& v) {
        take_slot(strand, v.lo);
        if (v.peer_in >= 0) emit(strand, v.lo, kRecvAct, v.peer_in);
        for (int id : m.plan.fwd_seq) emit(strand, v.lo, id);
        for (int l = v.lo + 1; l < v.hi; ++l) forward_layer(strand, l);
        if (v.peer_out >= 0) emit(strand, v.hi - 1, kSendAct, v.peer_out);
    }
    // backward span: mirror of the forward span (layers L-1-k for k in [lo, hi))
    void bwd_visit(int strand, const Visit& v, bool last_strand) {
        const int L = m.cfg.layers;
        const int top = L - 1 - v.lo, bottom = L - v.hi;
        if (v.peer_in >= 0) emit(strand, top, kRecvGrad, v.peer_in);
        for (int l = top; l >= bottom; --l) {
            backward_layer(strand, l);
            if (last_strand) emit_opt(strand, l);
        }
        if (v.peer_out >= 0) emit(strand, bottom, kSendGrad, v.peer_out);
    }
    void si_visit(int fs, int bs, const Visit& v, const weft::OverlapTable& tbl, bool relaxed) {
        const int L = m.cfg.layers;
        if (v.peer_in >= 0) {
            // the forward strand's first slot is taken by its first layer pair
            emit(bs, L - 1 - v.lo, kRecvGrad, v.peer_in);
        }
        for (int k = v.lo; k < v.hi; ++k) {
            if (k == v.lo && v.peer_in >= 0) pending_recv_act = {fs, v.peer_in};
            si_layer_pair(fs, k, bs, L - 1 - k, tbl, relaxed);
        }
        if (v.peer_out >= 0) {
            emit(fs, v.hi - 1, kSendAct, v.peer_out);
            emit(bs, L - v.hi, kSendGrad, v.peer_out);
        }
    }
    std::pair<int, int> pending_recv_act{-1, -1};  // (strand, peer) to receive right after a slot take
};

}  // namespace

int lower_ops(Model& m, int mode) {
    const int L = m.cfg.layers, mb = m.cfg.micro_batches;
    weft::OverlapTable tbl = weft::synth_profile(weft::ProfileArchetype::nvlink_h100).overlap;
    if (!m.plan_overlap.entries.empty()) tbl = m.plan_overlap;
    if (mode == 4 && n_slots(m) < L + 2)
        return set_error(DH_ERR_CONFIG, "mode 4 (deferred weight gradients) needs dh_model_cfg.slots >= layers + 2");
    Lowering lw(m);
    lw.prog.mode = mode;
    try {
        if (mode == 1) {
            for (int s = 0; s < mb; ++s) {
                lw.barrier();
                for (int l = 0; l < L; ++l) lw.forward_layer(s, l);
                for (int l = L - 1; l >= 0; --l) {
                    lw.backward_layer(s, l);
                    if (s == mb - 1) lw.emit_opt(s, l);
                }
            }
        } else if (mode == 3) {
            const int p = m.cfg.pp_size, d = m.cfg.pp_rank;
            if (L % 2 || m.cfg.split != (d + 1 < p ? L / 2 : 0))
                return set_error(DH_ERR_CONFIG, "w_pipeline: a stage holds an even number of layers, split at L/2 "
                                                "except on the last stage");
            const weft::PipelineSchedule ws = weft::schedule_w_pipeline(mb, p, weft::BlockDurations{});
            for (const auto& blk : ws.blocks) {
                if (blk.device != d) continue;
                lw.barrier();
                const auto v = lw.visit_of(blk);
                if (blk.kind == weft::BlockKind::F) {
                    lw.fwd_visit(*blk.fwd_mb - 1, v);
                } else if (blk.kind == weft::BlockKind::B) {
                    lw.bwd_visit(*blk.bwd_mb - 1, v, *blk.bwd_mb == mb);
                } else {
                    lw.si_visit(*blk.fwd_mb - 1, *blk.bwd_mb - 1, v, tbl, false);
                }
            }
        } else {
            // The block order is the reference W schedule on one stage
            // (schedule_w_pipeline(m, 1): F_1 | SI(F_{i+1}, B_i) ... | B_m, every
            // visit spanning the whole layer stack); only its order is used.
            const weft::PipelineSchedule ws = weft::schedule_w_pipeline(mb, 1, weft::BlockDurations{});
            for (const auto& blk : ws.blocks) {
                lw.barrier();
                if (blk.kind == weft::BlockKind::F) {
                    for (int l = 0; l < L; ++l) lw.forward_layer(*blk.fwd_mb - 1, l);
                } else if (blk.kind == weft::BlockKind::B) {
                    // mode 4: the lone strand defers each layer's attention weight
                    // gradients into the next layer, so that layer's AdamW follows
                    // the next layer's backward
                    const bool last_strand = *blk.bwd_mb == mb;
                    lw.lone_block = true;  // (no forward strand takes slots here: no extra slot needed)
                    const bool lag = lw.lone_defers();
                    for (int l = L - 1; l >= 0; --l) {
                        lw.backward_layer_dag(*blk.bwd_mb - 1, l);
                        if (last_strand && !lag) lw.emit_opt(mb - 1, l);
                        if (last_strand && lag && l + 1 < L) lw.emit_opt(mb - 1, l + 1);
                    }
                    if (lw.deferred.strand >= 0) {
                        lw.flush_deferred();
                        lw.strand_last[*blk.bwd_mb - 1] = lw.lane_last[0];  // AdamW(0) follows them
                    }
                    if (last_strand && lag) lw.emit_opt(mb - 1, 0);
                    lw.lone_block = false;
                } else {
                    lw.defer_wgrads = mode == 4;
                    for (int k = 0; k < L; ++k)
                        lw.si_layer_pair(*blk.fwd_mb - 1, k, *blk.bwd_mb - 1, L - 1 - k, tbl, mode == 2 || mode == 4);
                    lw.flush_deferred();  // the block's last pair: nothing to hide them under
                    lw.defer_wgrads = false;
                }
            }
        }
    } catch (const std::exception& e) {
        return set_error(DH_ERR_CONFIG, std::string("lowering: ") + e.what());
    }
    if (lw.free_slots.size() != static_cast<std::size_t>(n_slots(m)))
        return set_error(DH_ERR_OTHER, "lowering: activation slots leaked");
    m.prog_has_opt = lw.has_opt;
    m.peak_slots = lw.peak_slots;
    m.y_slot.assign(mb, -1);
    for (int s = 0; s < mb; ++s) m.y_slot[s] = lw.slot_of[s][L - 1];
    m.prog = std::move(lw.prog);
    return DH_OK;
}

int lower_program(Model& m, int mode) {
    RT_TRY(lower_ops(m, mode));
    // one event per op that some later op waits on
    for (auto e : m.events)
        if (e) cudaEventDestroy(e);
    m.events.assign(m.prog.ops.size(), nullptr);
    std::vector<char> needed(m.prog.ops.size(), 0);
    for (const auto& o : m.prog.ops)
        for (int w : o.waits) needed[w] = 1;
    RT_CUDA(cudaSetDevice(m.ctx->device));
    for (std::size_t i = 0; i < needed.size(); ++i) {
        if (needed[i]) RT_CUDA(cudaEventCreateWithFlags(&m.events[i], cudaEventDisableTiming));
    }
    if (m.graph) {
        cudaGraphExecDestroy(m.graph);
        m.graph = nullptr;
    }
    return DH_OK;
}

namespace {

// DH_OP_TIMES=<file> (eager runs only): CUDA events around every op, dumped
// as JSON lines (op, strand, layer, node, lane, start/end ms from the first op)
// after the program — the on-device timeline tools/op_timeline.py analyses.
struct OpTimes {
    std::vector<cudaEvent_t> ev;  // 2 per op
};

int issue(Model& m, OpTimes* ot = nullptr) {
    Ctx& c = *m.ctx;
    std::map<int, std::size_t> probe;  // node -> next probe slot
    static const bool trace = std::getenv("DH_TRACE") != nullptr;
    for (std::size_t i = 0; i < m.prog.ops.size(); ++i) {
        const Op& o = m.prog.ops[i];
        cudaStream_t s = c.lane[o.lane];
        for (int w : o.waits) RT_CUDA(cudaStreamWaitEvent(s, m.events[w], 0));
        auto pe = m.probe_events.find(o.node);
        std::pair<cudaEvent_t, cudaEvent_t>* pr = nullptr;
        if (pe != m.probe_events.end() && probe[o.node] < pe->second.size()) pr = &pe->second[probe[o.node]++];
        // External records stay real timing events inside a captured graph.
        if (pr) RT_CUDA(cudaEventRecordWithFlags(pr->first, s, cudaEventRecordExternal));
        if (trace) std::fprintf(stderr, "[dh] op %zu strand %d layer %d node %d lane %d\n", i, o.strand, o.layer, o.node, o.lane);
        if (ot) RT_CUDA(cudaEventRecord(ot->ev[2 * i], s));
        RT_TRY(launch_node(m, o, s));
        if (ot) RT_CUDA(cudaEventRecord(ot->ev[2 * i + 1], s));
        if (trace) {
            const cudaError_t e = cudaStreamSynchronize(s);
            std::fprintf(stderr, "[dh]   done: %s\n", cudaGetErrorString(e));
        }
        if (pr) RT_CUDA(cudaEventRecordWithFlags(pr->second, s, cudaEventRecordExternal));
        if (m.events[i]) RT_CUDA(cudaEventRecord(m.events[i], s));
    }
    return DH_OK;
}

// Fork lanes 1..2 off lane 0, run, join back into lane 0.
int issue_forked(Model& m, OpTimes* ot = nullptr) {
    Ctx& c = *m.ctx;
    if (!m.fork_join[0]) {
        for (auto& e : m.fork_join) RT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    RT_CUDA(cudaEventRecord(m.fork_join[0], c.lane[0]));
    for (int l = 1; l < kLanes; ++l) RT_CUDA(cudaStreamWaitEvent(c.lane[l], m.fork_join[0], 0));
    RT_TRY(issue(m, ot));
    for (int l = 1; l < kLanes; ++l) {
        RT_CUDA(cudaEventRecord(m.fork_join[l], c.lane[l]));
        RT_CUDA(cudaStreamWaitEvent(c.lane[0], m.fork_join[l], 0));
    }
    return DH_OK;
}

}  // namespace

int run_program(Model& m, bool use_graph) {
    if (m.prog.ops.empty()) return set_error(DH_ERR_CONFIG, "no program: call dh_model_set_plan first");
    RT_CUDA(cudaSetDevice(m.ctx->device));
    // A failure left pending by another library (e.g. the caller's framework)
    // would otherwise be reported against our first kernel launch.
    const cudaError_t pending = cudaGetLastError();
    if (pending != cudaSuccess) {
        std::fprintf(stderr, "[dh] cleared pending CUDA error before run_program: %s\n",
                     cudaGetErrorString(pending));
    }
    const bool capturable = !m.ctx->comm || m.ctx->comm->capturable();
    if (const char* path = std::getenv("DH_OP_TIMES"); path && !use_graph) {
        OpTimes ot;
        ot.ev.assign(2 * m.prog.ops.size(), nullptr);
        for (auto& e : ot.ev) RT_CUDA(cudaEventCreate(&e));
        const int rc = issue_forked(m, &ot);
        if (rc == DH_OK) {
            RT_CUDA(cudaStreamSynchronize(m.ctx->lane[0]));
            if (FILE* f = std::fopen(path, "w")) {
                for (std::size_t i = 0; i < m.prog.ops.size(); ++i) {
                    float a = 0.f, b = 0.f;
                    cudaEventElapsedTime(&a, ot.ev[0], ot.ev[2 * i]);
                    cudaEventElapsedTime(&b, ot.ev[0], ot.ev[2 * i + 1]);
                    const Op& o = m.prog.ops[i];
                    std::fprintf(f, "{\"op\": %zu, \"strand\": %d, \"layer\": %d, \"node\": %d, \"lane\": %d, "
                                    "\"capped\": %d, \"start_ms\": %.6f, \"end_ms\": %.6f}\n",
                                 i, o.strand, o.layer, o.node, o.lane, o.capped ? 1 : 0, a, b);
                }
                std::fclose(f);
            }
        }
        for (auto e : ot.ev) cudaEventDestroy(e);
        return rc;
    }
    if (!use_graph || !capturable) return issue_forked(m);
    if (!m.graph) {
        cudaStream_t s0 = m.ctx->lane[0];
        RT_CUDA(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
        const int rc = issue_forked(m);
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(s0, &g);
        if (rc != DH_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        RT_CUDA(e);
        const cudaError_t ie = cudaGraphInstantiate(&m.graph, g, 0);
        cudaGraphDestroy(g);
        RT_CUDA(ie);
    }
    RT_CUDA(cudaGraphLaunch(m.graph, m.ctx->lane[0]));
    return DH_OK;
}

// node < 0 clears every probe; otherwise adds `node` to the probed set.
int set_probe(Model& m, int node) {
    if (node < 0) {
        for (auto& [n, v] : m.probe_events)
            for (auto& pr : v) {
                cudaEventDestroy(pr.first);
                cudaEventDestroy(pr.second);
            }
        m.probe_events.clear();
        m.probe_nodes.clear();
    } else if (std::find(m.probe_nodes.begin(), m.probe_nodes.end(), node) == m.probe_nodes.end()) {
        m.probe_nodes.push_back(node);
    }
    if (m.graph) {
        cudaGraphExecDestroy(m.graph);
        m.graph = nullptr;
    }
    if (node < 0) return DH_OK;
    RT_CUDA(cudaSetDevice(m.ctx->device));
    auto& v = m.probe_events[node];
    for (auto& pr : v) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    v.clear();
    for (const auto& o : m.prog.ops) {
        if (o.node != node) continue;
        std::pair<cudaEvent_t, cudaEvent_t> pr{};
        RT_CUDA(cudaEventCreate(&pr.first));
        RT_CUDA(cudaEventCreate(&pr.second));
        v.push_back(pr);
    }
    return DH_OK;
}

// node < 0: the first probed node
int read_probe(Model& m, int node, double* total_ms, int* count) {
    if (node < 0 && !m.probe_nodes.empty()) node = m.probe_nodes.front();
    double sum = 0.0;
    int n = 0;
    auto it = m.probe_events.find(node);
    if (it != m.probe_events.end()) {
        for (auto& pr : it->second) {
            float ms = 0.f;
            RT_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
            sum += ms;
        }
        n = static_cast<int>(it->second.size());
    }
    *total_ms = sum;
    *count = n;
    return DH_OK;
}

}  // namespace dh
