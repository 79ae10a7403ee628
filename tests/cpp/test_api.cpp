// The C++ host API (include/mctune_b200.hpp) through the reference-style
// drop-in headers (include/compat/mctune/*.hpp): written against `mctune::`
// exactly as a caller of the reference library would, run on a B200.
#define MINI_DOCTEST_MAIN
#include "doctest.h"

#include <mctune/explore.hpp>
#include <mctune/model.hpp>
#include <mctune/search.hpp>

using namespace mctune;

namespace {
const PlatformConfig kPlat{1, 1, 4, 4};
}

TEST_CASE("launch shapes and the configuration space") {
    const LaunchPlan p = derive_launch(kPlat, 1024, {16, 32});
    CHECK(p == LaunchPlan{2, 1, 1, 4, 4});
    CHECK(enumerate_configs(1024).size() == 81);
    CHECK_THROWS_AS(derive_launch(PlatformConfig{1, 1, 3, 4}, 8, {2, 2}), ConfigError);
    CHECK_THROWS_AS(ProblemSpec::abstract(12), ConfigError);
}

TEST_CASE("paper Table 1: size 8 on (1,1,4,4) tunes to 44 at (4,4)") {
    const ProblemSpec problem = ProblemSpec::abstract(8);
    const TuneResult r = bisect_min_time(kPlat, problem, 100, ExploreLimits{});
    CHECK(r.t_min == 44);
    CHECK(r.params == TuningParams{4, 4});
    CHECK(r.proven);
    CHECK(r.trace.final_time == 44);
    CHECK(r.method == TuneMethod::Bisect);
    CHECK(replay(kPlat, problem, r.trace).time == 44);
    CHECK(extract_params(kPlat, problem, r.trace).time == 44);
    const Verdict below = check_overtime(kPlat, problem, 43, ExploreLimits{});
    CHECK_FALSE(below.violated);
    CHECK(below.exhaustive);
    CHECK_THROWS_AS(bisect_min_time(kPlat, problem, 43, ExploreLimits{}), ConfigError);
    ExploreLimits bitstate;
    bitstate.mode = ExploreLimits::Mode::Bitstate;
    CHECK_THROWS_AS(bisect_min_time(kPlat, problem, 100, bitstate), ConfigError);
}

TEST_CASE("tune from the estimated bound: size 64") {
    const ProblemSpec problem = ProblemSpec::abstract(64);
    const Tick est = estimate_initial_time(kPlat, problem, 1);
    const TuneResult r = tune(kPlat, problem, 1);
    CHECK(r.t_ini == est);
    CHECK(r.t_min == 324);
    CHECK(r.params == TuningParams{4, 32});
    CHECK(r.proven);
    CHECK(r.first_trail_optimality() > 0.0);
    CHECK(r.first_trail_optimality() <= 1.0);
    const auto rows = exhaustive_sweep(kPlat, problem);
    CHECK(rows.front().time == r.t_min);
}

TEST_CASE("every schedule of a configuration ends at the lock-step time") {
    const ProblemSpec problem = ProblemSpec::abstract(16);
    for (const auto& cfg : enumerate_configs(16)) {
        std::vector<Transition> tr;
        const RunOutcome rr = run(kPlat, problem, cfg, SchedPolicy::RoundRobin, 0, &tr);
        const RunOutcome sr = run(kPlat, problem, cfg, SchedPolicy::SeededRandom, 7);
        CHECK(rr.time == sr.time);
        CHECK(static_cast<long long>(tr.size()) == rr.transitions);
        const ExploreResult ex = explore_machine(kPlat, problem, cfg);
        CHECK(ex.complete);
        CHECK(ex.min_time == rr.time);
        CHECK(ex.max_time == rr.time);
        CHECK(ex.deadlocks == 0);
    }
}

TEST_CASE("minimum kernel: infeasible rows, result and replay") {
    const ProblemSpec problem = ProblemSpec::minimum(16);
    const auto rows = exhaustive_sweep(kPlat, problem);
    REQUIRE(rows.size() == 9);
    int flagged = 0;
    for (const auto& r : rows) flagged += !r.ok && r.note == "infeasible";
    CHECK(flagged == 3);
    CHECK(rows.front().time == 23);
    std::vector<Transition> tr;
    const RunOutcome o = run(kPlat, problem, {4, 4}, SchedPolicy::RoundRobin, 0, &tr);
    REQUIRE(o.result.has_value());
    CHECK(*o.result == 1);  // glob[0] = min of size - i
    Trace t{tr, o.time, {4, 4}, o.transitions};
    CHECK(replay(kPlat, problem, t).time == o.time);
    CHECK(!trace_to_text(kPlat, problem, t).empty());
    t.transitions.pop_back();
    CHECK_THROWS_AS(replay(kPlat, problem, t), CorruptTrace);
}

TEST_CASE("swarm agrees with bisection at desk scale") {
    const ProblemSpec problem = ProblemSpec::abstract(8);
    std::vector<Trace> trails;
    const TuneResult s = swarm_min_time(kPlat, problem, 2, ExploreLimits{}, 7, &trails);
    CHECK(s.t_min == 44);
    CHECK(s.params == TuningParams{4, 4});
    CHECK_FALSE(s.proven);
    CHECK(replay(kPlat, problem, s.trace).time == 44);
    CHECK(!trails.empty());
    const auto ranked = rank_trails(trails);
    CHECK(ranked.front().time == 44);
    const TuneResult again = swarm_min_time(kPlat, problem, 2, ExploreLimits{}, 7);
    CHECK(again.trace.transitions == s.trace.transitions);
    CHECK_THROWS_AS(swarm_min_time(kPlat, problem, 0, ExploreLimits{}, 1), ConfigError);
}

TEST_CASE("tuning-space argmin: the reference's space and a generalised one") {
    const ProblemSpec problem = ProblemSpec::abstract(64);
    const SpaceResult r = mctune_b200::space_argmin(mctune_b200::Space::reference(kPlat, problem));
    CHECK(r.time == 324);
    CHECK(r.params == TuningParams{4, 32});
    CHECK(r.platform == kPlat);
    mctune_b200::Space g;
    g.size = 1024;
    g.gmt = 4;
    g.nd_hi = 160000;
    g.nu_hi = 64;
    g.log2np_lo = 0;
    g.log2np_hi = 9;
    CHECK(g.count() == 8294400000ull);
    const SpaceResult w = mctune_b200::space_argmin(g, 0, 1000000000ull);
    CHECK(w.time == 5124);
    CHECK(w.index == 92160000ull);
    CHECK(w.params == TuningParams{512, 512});
}

TEST_CASE("swarm workers are deterministic per seed and sound (test_explore.cpp:112-143)") {
    const ProblemSpec problem = ProblemSpec::abstract(8);
    ExploreLimits limits;
    limits.mode = ExploreLimits::Mode::Bitstate;
    CHECK_THROWS_AS(swarm_worker(kPlat, problem, Property::non_termination(), 1, ExploreLimits{}),
                    ConfigError);
    const auto a = swarm_worker(kPlat, problem, Property::non_termination(), 5, limits);
    const auto b = swarm_worker(kPlat, problem, Property::non_termination(), 5, limits);
    REQUIRE(a.size() == b.size());
    CHECK(a.size() == 4);  // every feasible configuration ends at one time
    for (std::size_t i = 0; i < a.size(); ++i) {
        CHECK(a[i].final_time == b[i].final_time);
        CHECK(a[i].params == b[i].params);
        CHECK(a[i].transitions == b[i].transitions);
    }
    for (std::uint64_t seed : {1ull, 2ull}) {
        ExploreStats st;
        const auto traces = swarm_worker(kPlat, problem, Property::over_time(44), seed, limits, &st);
        // (2,4), (4,4) and (4,2) all finish at 44 (the sweep's rows), (2,2) at 88
        CHECK(traces.size() == 3);
        CHECK(st.configs_explored == 4);
        for (const auto& t : traces) {
            CHECK(t.final_time <= 44);
            CHECK(t.params != TuningParams{2, 2});
            CHECK(replay(kPlat, problem, t).time == t.final_time);
        }
    }
}

TEST_CASE("non-termination counterexamples enumerate terminating runs (test_explore.cpp:64-86)") {
    const ProblemSpec problem = ProblemSpec::abstract(8);
    ExploreLimits limits;
    const auto traces = check_nontermination(kPlat, problem, limits);
    REQUIRE(traces.size() == 4);
    Tick best = traces.front().final_time;
    std::vector<TuningParams> seen;
    for (const auto& t : traces) {
        best = std::min(best, t.final_time);
        if (std::find(seen.begin(), seen.end(), t.params) == seen.end()) seen.push_back(t.params);
        CHECK(replay(kPlat, problem, t).time == t.final_time);
    }
    CHECK(best == 44);
    CHECK(seen.size() == 4);
    CHECK(traces.front().params == TuningParams{4, 4});  // largest-first
    limits.max_depth = 1;
    CHECK(check_nontermination(kPlat, problem, limits).empty());
}

TEST_CASE("check_nontermination with several terminal states per configuration") {
    // (3,1,1,1) minimum size 16: host re-arming on three devices; the reference's
    // traces in DFS order (tests/golden/nonterm_multi.json)
    const PlatformConfig plat{3, 1, 1, 1};
    const ProblemSpec problem = ProblemSpec::minimum(16);
    ExploreStats stats;
    const auto traces = check_nontermination(plat, problem, ExploreLimits{}, &stats);
    REQUIRE(traces.size() == 25);
    CHECK(traces[0].params == TuningParams{8, 2});
    CHECK(traces[0].final_time == 17);
    CHECK(traces[0].steps == 79);
    CHECK(traces[1].params == TuningParams{4, 4});
    CHECK(traces[1].steps == 71);
    CHECK(traces[2].final_time == 9);
    CHECK(traces[3].steps == 83);
    CHECK(stats.states_visited == 32778);
    CHECK(stats.transitions_applied == 85370);
    CHECK(stats.max_depth_reached == 104);
    for (const auto& t : traces) CHECK(replay(plat, problem, t).time == t.final_time);
}

TEST_CASE("ExploreLimits::max_depth cuts the DFS") {
    const PlatformConfig plat{3, 1, 1, 1};
    const ProblemSpec problem = ProblemSpec::minimum(16);
    ExploreLimits limits;
    limits.max_depth = 67;
    const Verdict v = check_overtime(plat, problem, 17, limits);
    CHECK(v.violated);
    CHECK_FALSE(v.exhaustive);
    CHECK(v.stats.states_visited == 540);
    REQUIRE(v.trace.has_value());
    CHECK(v.trace->params == TuningParams{2, 8});
    CHECK(v.trace->steps == 67);
    const TuneResult r = tune(plat, problem, 1, limits);
    CHECK(r.t_min == 17);  // 9 without the cap
    CHECK(r.params == TuningParams{2, 8});
    CHECK_FALSE(r.proven);
    CHECK(r.stats.states_visited_total == 30165);
    limits.max_depth = 0;
    CHECK_THROWS_AS(check_overtime(plat, problem, 17, limits), ConfigError);
}

TEST_CASE("a binding visited cap moves the counterexample") {
    ExploreLimits limits;
    limits.max_states = 300;
    const TuneResult r = tune(kPlat, ProblemSpec::abstract(16), 1, limits);
    CHECK(r.t_min == 84);
    CHECK(r.params == TuningParams{2, 8});  // (4, 8) without the cap
    CHECK(r.stats.states_visited_total == 20980);
}

TEST_CASE("explore_machine with hooks agrees with the batched sweep, caps included") {
    // the DFS-order walk (mctb_machine_states) and the sweep's statistics
    // (mctb_explore, pinned to the reference) on every configuration, with a
    // binding visited cap and a depth cap
    const PlatformConfig plats[] = {{1, 1, 4, 4}, {2, 1, 2, 4}};
    for (const auto& plat : plats) {
        const ProblemSpec problem = ProblemSpec::abstract(16);
        for (long long cap : {5'000'000LL, 500LL}) {
            for (long long depth : {4'000'000LL, 60LL}) {
                ExploreLimits limits;
                limits.max_states = cap;
                limits.max_depth = depth;
                const auto cfgs = enumerate_configs(problem.size);
                const auto want = explore_configs(plat, problem, cfgs, limits);
                for (std::size_t k = 0; k < cfgs.size(); ++k) {
                    Machine m(plat, problem, cfgs[k]);
                    ExploreStats st;
                    long long on_state = 0, on_term = 0;
                    ExploreHooks hooks;
                    hooks.on_state = [&](const Machine&, const MachineState&) { ++on_state; };
                    hooks.on_terminal = [&](const Machine& mm, const MachineState& s,
                                            const std::vector<Transition>& path) {
                        ++on_term;
                        // the path replays to this terminal state
                        CHECK(replay(mm.platform, mm.problem,
                                     Trace{path, s.time, mm.params,
                                           static_cast<long long>(path.size())})
                                  .time == s.time);
                        return true;
                    };
                    const bool complete = explore_machine(m, limits, st, hooks);
                    CHECK(complete == want[k].complete);
                    CHECK(st.states_visited == want[k].stats.states_visited);
                    CHECK(on_state == st.states_visited);
                    CHECK(st.transitions_applied == want[k].stats.transitions_applied);
                    CHECK(st.max_depth_reached == want[k].stats.max_depth_reached);
                    if (want[k].complete) CHECK(on_term == want[k].terminal_states);
                }
            }
        }
    }
}
