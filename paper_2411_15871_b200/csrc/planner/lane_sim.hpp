// Internal: the three-lane co-execution simulator shared by
// segment_pair_cost() (public API) and the plan search's memoised cost
// function. One implementation, so both paths produce identical doubles.
//
// Rules restated from /root/reference/proj/src/overlap_profile.cpp:129-222:
//   * each strand runs its ops in order; a lane holds one op at a time;
//   * when several fronts can start, the smaller (release time, solo time,
//     class id) starts first, strand 0 winning exact ties;
//   * two co-running ops both progress at 1/((2-e)(1+slowdown)), where e is
//     the pair's OEF clamped to [0,1], less launch_overhead_frac (floored at
//     0) when either op sits on a communication lane;
//   * time advances to the next completion; an op finishes when
//     remaining/rate <= dt, otherwise remaining -= rate*dt.
#pragma once

#include <algorithm>
#include <array>
#include <cstddef>
#include <limits>
#include <tuple>
#include <utility>
#include <vector>

#include "weft/overlap_profile.hpp"

namespace weft::detail {

struct SimOp {
    double t_us;  // resolved solo time
    Lane lane;
    OperatorClass cls;
};

// `raw_oef(a, b)` returns the table OEF for the pair (throws when missing).
// `trace`, when given, receives (strand, op index) in dispatch (start) order —
// the B200 executor lowers a plan step to lane-stream launches in this order;
// `spans` (with `trace`) receives each traced op's simulated (start, end).
// Neither output changes the arithmetic.
template <class RawOef>
SegmentCost simulate_lanes(const SimOp* ops_a, std::size_t n_a, const SimOp* ops_b,
                           std::size_t n_b, double slowdown, double launch_frac,
                           RawOef&& raw_oef,
                           std::vector<std::pair<int, std::size_t>>* trace = nullptr,
                           std::vector<std::pair<double, double>>* spans = nullptr) {
    struct Front {
        const SimOp* ops;
        std::size_t n;
        std::size_t next = 0;
        const SimOp* cur = nullptr;
        double remaining = 0.0;
        double release = 0.0;
        bool busy = false;
        std::size_t span = 0;  // index of the current op in *spans
    };
    std::array<Front, 2> fr{Front{ops_a, n_a}, Front{ops_b, n_b}};
    std::array<int, 3> owner{-1, -1, -1};
    SegmentCost cost;
    double clock = 0.0;

    auto start_ready = [&]() {
        for (;;) {
            int chosen = -1;
            for (int s = 0; s < 2; ++s) {
                Front& f = fr[s];
                if (f.busy || f.next >= f.n) continue;
                const SimOp& cand = f.ops[f.next];
                if (owner[static_cast<int>(cand.lane)] != -1) continue;
                if (chosen < 0) {
                    chosen = s;
                    continue;
                }
                const Front& g = fr[chosen];
                const SimOp& held = g.ops[g.next];
                if (std::make_tuple(f.release, cand.t_us, static_cast<int>(cand.cls)) <
                    std::make_tuple(g.release, held.t_us, static_cast<int>(held.cls))) {
                    chosen = s;
                }
            }
            if (chosen < 0) return;
            Front& f = fr[chosen];
            if (trace) trace->emplace_back(chosen, f.next);
            if (trace && spans) {
                f.span = spans->size();
                spans->emplace_back(clock, clock);
            }
            f.cur = &f.ops[f.next++];
            f.remaining = f.cur->t_us;
            f.busy = true;
            owner[static_cast<int>(f.cur->lane)] = chosen;
            if (f.remaining <= 0.0) {
                f.busy = false;
                owner[static_cast<int>(f.cur->lane)] = -1;
                f.release = clock;
            }
        }
    };

    start_ready();
    while (fr[0].busy || fr[1].busy) {
        double r0 = 1.0, r1 = 1.0;
        if (fr[0].busy && fr[1].busy) {
            double e = std::clamp(raw_oef(*fr[0].cur, *fr[1].cur), 0.0, 1.0);
            if (fr[0].cur->lane != Lane::compute || fr[1].cur->lane != Lane::compute) {
                e = std::max(0.0, e - launch_frac);
            }
            r0 = r1 = 1.0 / ((2.0 - e) * (1.0 + slowdown));
        }
        double dt = std::numeric_limits<double>::infinity();
        if (fr[0].busy) dt = std::min(dt, fr[0].remaining / r0);
        if (fr[1].busy) dt = std::min(dt, fr[1].remaining / r1);
        for (int s = 0; s < 2; ++s) {
            Front& f = fr[s];
            if (!f.busy) continue;
            const double r = s == 0 ? r0 : r1;
            cost.lane_busy_us[static_cast<int>(f.cur->lane)] += dt;
            if (f.remaining / r <= dt) {
                if (trace && spans) (*spans)[f.span].second = clock + dt;
                f.remaining = 0.0;
                f.busy = false;
                owner[static_cast<int>(f.cur->lane)] = -1;
                f.release = clock + dt;
            } else {
                f.remaining -= r * dt;
            }
        }
        clock += dt;
        start_ready();
    }
    cost.p_us = clock;
    return cost;
}

}  // namespace weft::detail
