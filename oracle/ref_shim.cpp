// TEST INFRASTRUCTURE ONLY — never part of the product path.
//
// extern "C" shim over the reference's own C++ core (mctune, compiled from
// /root/reference/proj/src/{model,kernel,machine,explore,search}.cpp by
// oracle/Makefile into oracle/_ref/libmctune_ref.so).  It lets the tests,
// the golden-vector generator (tests/golden/make_golden.py) and bench.py's
// reference arm run the UNMODIFIED reference algorithm.  Nothing here
// re-implements reference behaviour except trace_to_text, which the
// reference keeps in report.cpp (needs the un-vendored nlohmann/json, so
// report.cpp itself cannot be compiled here); the rendering below follows
// report.cpp:82-97 using only Machine::label / role_of / to_string.
//
// Transition exchange format: 4 x int32 per transition
//   [actor, peer, op, arg]   (peer 0xffff = none; op = mctune::Op ordinal)
// Return codes: 0 ok, 1 ModelBug, 2 ConfigError, 3 CorruptTrace, 4 other.

#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "mctune/explore.hpp"
#include "mctune/machine.hpp"
#include "mctune/search.hpp"

using namespace mctune;

namespace {

thread_local std::string g_err;

PlatformConfig plat_of(const int* p) { return PlatformConfig{p[0], p[1], p[2], p[3]}; }

ProblemSpec problem_of(int size, int kernel, const int64_t* input) {
    if (kernel == 0) return ProblemSpec::abstract(size);
    std::vector<std::int64_t> in;
    if (input) in.assign(input, input + size);
    return ProblemSpec::minimum(size, std::move(in));
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const CorruptTrace& e) {
        g_err = e.what();
        return 3;
    } catch (const ModelBug& e) {
        g_err = e.what();
        return 1;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

void put_trace(const std::vector<Transition>& tr, int32_t* buf, long long cap, long long* len) {
    if (len) *len = static_cast<long long>(tr.size());
    if (!buf) return;
    const long long n = std::min<long long>(cap, static_cast<long long>(tr.size()));
    for (long long i = 0; i < n; ++i) {
        buf[4 * i + 0] = tr[static_cast<std::size_t>(i)].actor;
        buf[4 * i + 1] = tr[static_cast<std::size_t>(i)].peer;
        buf[4 * i + 2] = static_cast<int32_t>(tr[static_cast<std::size_t>(i)].op);
        buf[4 * i + 3] = tr[static_cast<std::size_t>(i)].arg;
    }
}

std::vector<Transition> get_trace(const int32_t* buf, long long len) {
    std::vector<Transition> out(static_cast<std::size_t>(len));
    for (long long i = 0; i < len; ++i) {
        Transition& t = out[static_cast<std::size_t>(i)];
        t.actor = static_cast<std::uint16_t>(buf[4 * i + 0]);
        t.peer = static_cast<std::uint16_t>(buf[4 * i + 1]);
        t.op = static_cast<Op>(buf[4 * i + 2]);
        t.arg = buf[4 * i + 3];
    }
    return out;
}

ExploreLimits limits_of(long long max_depth, long long max_states, int bitstate, double budget) {
    ExploreLimits l;
    if (max_depth > 0) l.max_depth = max_depth;
    if (max_states > 0) l.max_states = max_states;
    l.mode = bitstate ? ExploreLimits::Mode::Bitstate : ExploreLimits::Mode::Exact;
    l.wall_budget_secs = budget;
    return l;
}

// report.cpp:82-97 rendering, re-expressed over the public Machine API.
std::string render(const PlatformConfig& platform, const ProblemSpec& problem, const Trace& trace) {
    Machine m(platform, problem, trace.params);
    MachineState s = m.initial_state();
    std::ostringstream os;
    for (std::size_t i = 0; i < trace.transitions.size(); ++i) {
        const Transition& t = trace.transitions[i];
        s = m.apply(s, t);
        os << i << ' ' << t.actor << ' ' << to_string(m.role_of(t.actor)) << ' ' << m.label(t)
           << " time=" << s.time << '\n';
    }
    os << "FINAL time=" << s.time << " wg=" << trace.params.wg << " ts=" << trace.params.ts;
    if (problem.kernel == KernelKind::Minimum) os << " result=" << s.glob[0];
    os << '\n';
    return os.str();
}

long long put_text(const std::string& s, char* buf, long long cap) {
    if (buf && cap > 0) {
        const long long n = std::min<long long>(cap - 1, static_cast<long long>(s.size()));
        std::memcpy(buf, s.data(), static_cast<std::size_t>(n));
        buf[n] = 0;
    }
    return static_cast<long long>(s.size());
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// derive_launch (model.cpp:72-88): out = [wgs, nwd, nwu, nwe, all_nwe]
int ref_derive_launch(const int* plat, int size, int wg, int ts, int* out) {
    return guarded([&] {
        const LaunchPlan p = derive_launch(plat_of(plat), size, TuningParams{wg, ts});
        out[0] = p.wgs;
        out[1] = p.nwd;
        out[2] = p.nwu;
        out[3] = p.nwe;
        out[4] = p.all_nwe;
    });
}

// Machine::run (machine.cpp:788-825).  policy 0 = RoundRobin, 1 = SeededRandom.
// out = [time, steps, result(or INT64_MIN), process_count]
int ref_simulate(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                 int policy, uint64_t seed, int64_t* out, int32_t* trace, long long cap,
                 long long* trace_len) {
    return guarded([&] {
        Machine m(plat_of(plat), problem_of(size, kernel, input), TuningParams{wg, ts});
        std::vector<Transition> tr;
        const RunOutcome r = m.run(policy ? SchedPolicy::SeededRandom : SchedPolicy::RoundRobin,
                                   seed, trace ? &tr : nullptr);
        out[0] = r.time;
        out[1] = r.steps;
        out[2] = r.result ? *r.result : INT64_MIN;
        out[3] = m.process_count();
        if (trace) put_trace(tr, trace, cap, trace_len);
    });
}

// Fingerprints (machine.cpp:715) of every state along a run, initial state first.
int ref_run_fingerprints(const int* plat, int size, int kernel, const int64_t* input, int wg,
                         int ts, const int32_t* trace, long long len, uint64_t* out) {
    return guarded([&] {
        Machine m(plat_of(plat), problem_of(size, kernel, input), TuningParams{wg, ts});
        MachineState s = m.initial_state();
        out[0] = m.fingerprint(s);
        const auto tr = get_trace(trace, len);
        for (long long i = 0; i < len; ++i) {
            s = m.apply(s, tr[static_cast<std::size_t>(i)]);
            out[i + 1] = m.fingerprint(s);
        }
    });
}

// Canonical serialization of the initial state (machine.cpp:669-706).
long long ref_serialize_initial(const int* plat, int size, int kernel, const int64_t* input,
                                int wg, int ts, unsigned char* buf, long long cap) {
    long long n = -1;
    guarded([&] {
        Machine m(plat_of(plat), problem_of(size, kernel, input), TuningParams{wg, ts});
        const std::string s = m.serialize(m.initial_state());
        n = static_cast<long long>(s.size());
        if (buf) std::memcpy(buf, s.data(), static_cast<std::size_t>(std::min<long long>(n, cap)));
    });
    return n;
}

// Enabled transitions after replaying a prefix (machine.cpp:174-336).
int ref_enabled_after(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                      const int32_t* trace, long long len, int32_t* out, long long cap,
                      long long* n_out) {
    return guarded([&] {
        Machine m(plat_of(plat), problem_of(size, kernel, input), TuningParams{wg, ts});
        MachineState s = m.initial_state();
        const auto tr = get_trace(trace, len);
        for (const auto& t : tr) s = m.apply(s, t);
        put_trace(m.enabled(s), out, cap, n_out);
    });
}

// explore_machine (explore.cpp:86-165) over ONE configuration, every interleaving.
// out = [complete, states_visited, transitions_applied, max_depth_reached,
//        min_final_time, max_final_time, n_terminal_states, n_distinct_times]
int ref_explore(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                long long max_depth, long long max_states, int bitstate, int check_invariants,
                int64_t* out) {
    return guarded([&] {
        Machine m(plat_of(plat), problem_of(size, kernel, input), TuningParams{wg, ts});
        ExploreStats stats;
        long long n_term = 0;
        Tick lo = -1, hi = -1;
        std::vector<Tick> times;
        ExploreHooks hooks;
        if (check_invariants)
            hooks.on_state = [](const Machine& mm, const MachineState& s) { mm.check_invariants(s); };
        hooks.on_terminal = [&](const Machine&, const MachineState& s,
                                const std::vector<Transition>&) {
            ++n_term;
            lo = lo < 0 ? s.time : std::min(lo, s.time);
            hi = std::max(hi, s.time);
            if (std::find(times.begin(), times.end(), s.time) == times.end()) times.push_back(s.time);
            return true;
        };
        const bool complete =
            explore_machine(m, limits_of(max_depth, max_states, bitstate, 0.0), stats, hooks);
        out[0] = complete;
        out[1] = stats.states_visited;
        out[2] = stats.transitions_applied;
        out[3] = stats.max_depth_reached;
        out[4] = lo;
        out[5] = hi;
        out[6] = n_term;
        out[7] = static_cast<int64_t>(times.size());
    });
}

// explore_machine's discovery order (explore.cpp:86-165): FNV-1a 64 of every
// visited state, in on_state order, over its fields as int64 values in the order
// of the engine's flat state vector (include/mctune_b200.h, mctb_machine_*):
// time, nrp_work, all_nwe, fin, next_wg, host {pc, k}, clock, then counted
// device, unit, barrier and element records, glob and loc.
int ref_explore_order(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                      long long max_depth, long long max_states, uint64_t* hashes, long long cap,
                      long long* n) {
    return guarded([&] {
        Machine m(plat_of(plat), problem_of(size, kernel, input), TuningParams{wg, ts});
        ExploreStats stats;
        long long count = 0;
        ExploreHooks hooks;
        hooks.on_state = [&](const Machine&, const MachineState& s) {
            uint64_t h = 0xcbf29ce484222325ull;
            auto put = [&](int64_t v) {
                for (int b = 0; b < 8; ++b) {
                    h ^= static_cast<uint64_t>(v >> (8 * b)) & 0xffu;
                    h *= 0x100000001b3ull;
                }
            };
            put(s.time);
            put(s.nrp_work);
            put(s.all_nwe);
            put(s.fin);
            put(s.next_wg);
            put(static_cast<int64_t>(s.host.pc));
            put(s.host.k);
            put(static_cast<int64_t>(s.clock));
            put(static_cast<int64_t>(s.devices.size()));
            for (const auto& d : s.devices) {
                put(static_cast<int64_t>(d.pc));
                put(d.k);
                put(d.batch_base);
            }
            put(static_cast<int64_t>(s.units.size()));
            for (const auto& u : s.units) {
                put(static_cast<int64_t>(u.pc));
                put(u.k);
                put(u.nwg);
                put(u.sent);
                put(u.got_items);
                put(u.got_ends);
            }
            put(static_cast<int64_t>(s.barriers.size()));
            for (const auto& b : s.barriers) {
                put(static_cast<int64_t>(b.pc));
                put(b.count);
            }
            put(static_cast<int64_t>(s.pexes.size()));
            for (const auto& x : s.pexes) {
                put(static_cast<int64_t>(x.pc));
                put(static_cast<int64_t>(x.phase));
                put(x.cursor);
                put(x.busy_left);
                put(x.reported);
                put(x.nwg);
                put(x.iter);
            }
            put(static_cast<int64_t>(s.glob.size()));
            for (auto v : s.glob) put(v);
            put(static_cast<int64_t>(s.loc.size()));
            for (auto v : s.loc) put(v);
            if (count < cap) hashes[count] = h;
            ++count;
        };
        explore_machine(m, limits_of(max_depth, max_states, 0, 0.0), stats, hooks);
        *n = count;
    });
}

// check_overtime (explore.cpp:167-205).
// out = [violated, exhaustive, states_visited, max_depth_reached, transitions_applied,
//        configs_explored, configs_skipped, final_time, wg, ts, steps]
int ref_check_overtime(const int* plat, int size, int kernel, const int64_t* input, int64_t T,
                       long long max_depth, long long max_states, int bitstate, int64_t* out,
                       int32_t* trace, long long cap, long long* trace_len) {
    return guarded([&] {
        const Verdict v = check_overtime(plat_of(plat), problem_of(size, kernel, input), T,
                                         limits_of(max_depth, max_states, bitstate, 0.0));
        out[0] = v.violated;
        out[1] = v.exhaustive;
        out[2] = v.stats.states_visited;
        out[3] = v.stats.max_depth_reached;
        out[4] = v.stats.transitions_applied;
        out[5] = v.stats.configs_explored;
        out[6] = v.stats.configs_skipped;
        out[7] = v.trace ? v.trace->final_time : -1;
        out[8] = v.trace ? v.trace->params.wg : 0;
        out[9] = v.trace ? v.trace->params.ts : 0;
        out[10] = v.trace ? v.trace->steps : 0;
        if (v.trace && trace_len) put_trace(v.trace->transitions, trace, cap, trace_len);
        else if (trace_len) *trace_len = 0;
    });
}

// check_nontermination (explore.cpp:207-233): rows = [wg, ts, final_time, steps] per
// trace (up to cap_rows), traces concatenated into `trace` (4 ints per transition);
// out = [n_traces, states_visited, transitions_applied, max_depth_reached, limit_hit]
int ref_check_nontermination(const int* plat, int size, int kernel, const int64_t* input,
                             long long max_depth, long long max_states, int64_t* out,
                             int64_t* rows, long long cap_rows, int32_t* trace, long long cap,
                             long long* trace_len) {
    return guarded([&] {
        ExploreStats st;
        const auto traces = check_nontermination(plat_of(plat), problem_of(size, kernel, input),
                                                 limits_of(max_depth, max_states, 0, 0.0), &st);
        out[0] = static_cast<int64_t>(traces.size());
        out[1] = st.states_visited;
        out[2] = st.transitions_applied;
        out[3] = st.max_depth_reached;
        out[4] = st.limit_hit;
        std::vector<Transition> all;
        for (std::size_t i = 0; i < traces.size(); ++i) {
            if (static_cast<long long>(i) < cap_rows) {
                rows[4 * i] = traces[i].params.wg;
                rows[4 * i + 1] = traces[i].params.ts;
                rows[4 * i + 2] = traces[i].final_time;
                rows[4 * i + 3] = traces[i].steps;
            }
            all.insert(all.end(), traces[i].transitions.begin(), traces[i].transitions.end());
        }
        put_trace(all, trace, cap, trace_len);
    });
}

// estimate_initial_time (search.cpp:94-102)
int ref_estimate_initial_time(const int* plat, int size, int kernel, const int64_t* input,
                              uint64_t seed, int64_t* out) {
    return guarded([&] {
        *out = estimate_initial_time(plat_of(plat), problem_of(size, kernel, input), seed);
    });
}

// bisect_min_time (search.cpp:104-158).  t_hi <= 0 means estimate_initial_time(seed) first
// (the `tune` command flow, tools/main.cpp:119-128).
// out = [t_min, wg, ts, t_ini, proven, checks_run, states_visited_total, first_trail_time, steps]
int ref_tune(const int* plat, int size, int kernel, const int64_t* input, int64_t t_hi,
             uint64_t seed, long long max_depth, long long max_states, int64_t* out,
             int32_t* trace, long long cap, long long* trace_len) {
    return guarded([&] {
        const PlatformConfig p = plat_of(plat);
        const ProblemSpec prob = problem_of(size, kernel, input);
        if (t_hi <= 0) t_hi = estimate_initial_time(p, prob, seed);
        const TuneResult r = bisect_min_time(p, prob, t_hi, limits_of(max_depth, max_states, 0, 0.0));
        out[0] = r.t_min;
        out[1] = r.params.wg;
        out[2] = r.params.ts;
        out[3] = r.t_ini;
        out[4] = r.proven;
        out[5] = r.stats.checks_run;
        out[6] = r.stats.states_visited_total;
        out[7] = r.first_trail_time;
        out[8] = r.trace.steps;
        if (trace_len) put_trace(r.trace.transitions, trace, cap, trace_len);
    });
}

// exhaustive_sweep (search.cpp:212-244).  rows: [wg, ts, time, transitions, ok, note]
// note: 0 none, 1 infeasible, 2 deadlock.  Returns row count via *n_rows.
int ref_sweep(const int* plat, int size, int kernel, const int64_t* input, int64_t* rows,
              long long cap, long long* n_rows) {
    return guarded([&] {
        const auto rs = exhaustive_sweep(plat_of(plat), problem_of(size, kernel, input));
        *n_rows = static_cast<long long>(rs.size());
        for (std::size_t i = 0; i < rs.size() && static_cast<long long>(i) < cap; ++i) {
            rows[6 * i + 0] = rs[i].wg;
            rows[6 * i + 1] = rs[i].ts;
            rows[6 * i + 2] = rs[i].time;
            rows[6 * i + 3] = rs[i].transitions;
            rows[6 * i + 4] = rs[i].ok;
            rows[6 * i + 5] = rs[i].note == "infeasible" ? 1 : (rs[i].note == "deadlock" ? 2 : 0);
        }
    });
}

// replay (explore.cpp:283-300).  out = [final_time, result(or INT64_MIN)]
int ref_replay(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
               const int32_t* trace, long long len, int64_t final_time, int64_t* out) {
    return guarded([&] {
        Trace t;
        t.params = TuningParams{wg, ts};
        t.transitions = get_trace(trace, len);
        t.final_time = final_time;
        t.steps = len;
        const ProblemSpec prob = problem_of(size, kernel, input);
        const MachineState s = replay(plat_of(plat), prob, t);
        out[0] = s.time;
        out[1] = prob.kernel == KernelKind::Minimum ? s.glob[0] : INT64_MIN;
    });
}

// Trace text (report.cpp:82-97).  Returns the full text length; copies at most cap-1 bytes.
long long ref_trace_text(const int* plat, int size, int kernel, const int64_t* input, int wg,
                         int ts, const int32_t* trace, long long len, char* buf, long long cap) {
    long long n = -1;
    guarded([&] {
        Trace t;
        t.params = TuningParams{wg, ts};
        t.transitions = get_trace(trace, len);
        n = put_text(render(plat_of(plat), problem_of(size, kernel, input), t), buf, cap);
    });
    return n;
}

// swarm_min_time (search.cpp:160-210), for timing and for the >= bisection property.
// out = [t_min, wg, ts, t_ini, checks_run, states_visited_total, first_trail_time, steps]
int ref_swarm(const int* plat, int size, int kernel, const int64_t* input, int workers,
              double budget_secs, long long max_depth, uint64_t seed, int64_t* out) {
    return guarded([&] {
        const TuneResult r = swarm_min_time(plat_of(plat), problem_of(size, kernel, input), workers,
                                            limits_of(max_depth, 0, 1, budget_secs), seed);
        out[0] = r.t_min;
        out[1] = r.params.wg;
        out[2] = r.params.ts;
        out[3] = r.t_ini;
        out[4] = r.stats.checks_run;
        out[5] = r.stats.states_visited_total;
        out[6] = r.first_trail_time;
        out[7] = r.trace.steps;
    });
}

}  // extern "C"
