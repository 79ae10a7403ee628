// mctune_b200.hpp — the C++ host API of the B200 search engine.
//
// A header-only mirror of the reference library's public interface
// (/root/reference/proj/include/mctune/{model,explore,search}.hpp): the same
// type names, fields, function signatures, argument meanings and exception
// classes, implemented on the C ABI of include/mctune_b200.h (every model time
// is computed by sm_100a kernels; there is no CPU path — calls throw NoDevice
// without a B200).  Code written against `mctune::` compiles against this
// header through include/compat/mctune/*.hpp, which alias the namespace.
//
// Link: -L<repo>/paper_2305_09130_b200 -lmctune_b200 (C++20).
#ifndef MCTUNE_B200_HPP
#define MCTUNE_B200_HPP

#include <algorithm>
#include <functional>
#include <atomic>
#include <array>
#include <chrono>
#include <cstdint>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "mctune_b200.h"

namespace mctune_b200 {

/// Model time, in clock ticks (model.hpp:12).
using Tick = std::int64_t;

// ------------------------------------------------------------------ errors
/// Invalid user input (model.hpp:15-17).
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// Internal contract violation of the transition system (model.hpp:20-22).
struct ModelBug : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// A trace failed to replay (explore.hpp:14-17).
struct CorruptTrace : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// No sm_100 device is visible (the engine has no CPU path).
struct NoDevice : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// A GPU capacity limit (state packing, visited table) was exceeded.
struct LimitError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
    if (rc == MCTB_OK) return;
    const std::string msg = mctb_last_error() ? mctb_last_error() : "";
    switch (rc) {
        case MCTB_CONFIG_ERROR: throw ConfigError(msg);
        case MCTB_MODEL_BUG: throw ModelBug(msg);
        case MCTB_CORRUPT_TRACE: throw CorruptTrace(msg);
        case MCTB_NO_DEVICE: throw NoDevice(msg.empty() ? "no sm_100 device" : msg);
        case MCTB_LIMIT: throw LimitError(msg);
        default: throw std::runtime_error("CUDA error: " + msg);
    }
}
}  // namespace detail

// ------------------------------------------------------------------ model (model.hpp)
constexpr bool is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }

/// Exact log2 of a power of two (model.cpp:5-10).
inline int log2_exact(int v) {
    if (!is_pow2(v)) throw ConfigError("not a power of two: " + std::to_string(v));
    int k = 0;
    while ((1 << k) < v) ++k;
    return k;
}

/// Architecture constants of the abstract platform (model.hpp:33-40).
struct PlatformConfig {
    int nd = 1;
    int nu = 1;
    int np = 4;
    int gmt = 4;

    void validate() const {  // model.cpp:12-17
        if (nd < 1 || nu < 1 || np < 1 || gmt < 1)
            throw ConfigError("platform constants nd, nu, np, gmt must all be >= 1");
        if (!is_pow2(np)) throw ConfigError("np must be a power of two, got " + std::to_string(np));
    }
    bool operator==(const PlatformConfig&) const = default;
};

enum class KernelKind : std::uint8_t { Abstract, Minimum };

inline const char* to_string(KernelKind k) {
    return k == KernelKind::Abstract ? "abstract" : "minimum";
}

inline KernelKind kernel_kind_from_string(const std::string& s) {  // model.cpp:23-27
    if (s == "abstract") return KernelKind::Abstract;
    if (s == "minimum") return KernelKind::Minimum;
    throw ConfigError("unknown kernel kind '" + s + "' (expected abstract or minimum)");
}

/// The problem instance (model.hpp:48-58).
struct ProblemSpec {
    int size = 8;
    KernelKind kernel = KernelKind::Abstract;
    std::vector<std::int64_t> input;  // minimum kernel only, length == size

    static ProblemSpec abstract(int size) {
        ProblemSpec p;
        p.size = size;
        p.validate();
        return p;
    }
    /// Minimum kernel; empty input selects the default glob[i] = size - i.
    static ProblemSpec minimum(int size, std::vector<std::int64_t> input = {}) {
        ProblemSpec p;
        p.size = size;
        p.kernel = KernelKind::Minimum;
        if (input.empty() && size > 0)
            for (int i = 0; i < size; ++i) input.push_back(size - i);
        p.input = std::move(input);
        p.validate();
        return p;
    }
    void validate() const {  // model.cpp:51-60
        if (size < 4 || !is_pow2(size))
            throw ConfigError("size must be a power of two >= 4, got " + std::to_string(size));
        if (kernel == KernelKind::Minimum) {
            if (static_cast<int>(input.size()) != size)
                throw ConfigError("minimum kernel needs an input array of length size");
        } else if (!input.empty()) {
            throw ConfigError("abstract kernel takes no input array");
        }
    }
};

/// The two tuning parameters (model.hpp:61-66).
struct TuningParams {
    int wg = 0;
    int ts = 0;
    bool operator==(const TuningParams&) const = default;
};

/// Launch shape derived from (platform, size, params) (model.hpp:69-77).
struct LaunchPlan {
    int wgs = 0;
    int nwd = 0;
    int nwu = 0;
    int nwe = 0;
    int all_nwe = 0;
    bool operator==(const LaunchPlan&) const = default;
};

/// model.cpp:62-70
inline void validate_params(int size, const TuningParams& params) {
    const int hi = size / 2;
    if (!is_pow2(params.wg) || params.wg < 2 || params.wg > hi)
        throw ConfigError("wg must be a power of two in [2, size/2], got " + std::to_string(params.wg));
    if (!is_pow2(params.ts) || params.ts < 2 || params.ts > hi)
        throw ConfigError("ts must be a power of two in [2, size/2], got " + std::to_string(params.ts));
}

/// Listing-3 launch arithmetic (model.cpp:72-88), mctb_derive_launch.
inline LaunchPlan derive_launch(const PlatformConfig& platform, int size, const TuningParams& params) {
    const int plat[4] = {platform.nd, platform.nu, platform.np, platform.gmt};
    int out[5];
    detail::check(mctb_derive_launch(plat, size, params.wg, params.ts, out));
    return LaunchPlan{out[0], out[1], out[2], out[3], out[4]};
}

/// All (wg, ts) = (2^i, 2^j), i, j in [1, n-1], ascending (model.cpp:90-100).
inline std::vector<TuningParams> enumerate_configs(int size) {
    if (size < 4 || !is_pow2(size))
        throw ConfigError("size must be a power of two >= 4, got " + std::to_string(size));
    const int n = log2_exact(size);
    std::vector<TuningParams> out;
    for (int i = 1; i < n; ++i)
        for (int j = 1; j < n; ++j) out.push_back(TuningParams{1 << i, 1 << j});
    return out;
}

/// kernel.cpp:84-87: the minimum kernel needs wg * ts <= size.
inline bool config_feasible(const ProblemSpec& problem, const TuningParams& params) {
    return problem.kernel == KernelKind::Abstract || params.wg * params.ts <= problem.size;
}

// ------------------------------------------------------------------ kernel (kernel.hpp)
/// kernel.hpp:11-46: memory spaces and the symbolic operands of effects.
enum class MemSpace : std::uint8_t { Global, Local };

struct MemRef {
    enum class Base : std::uint8_t { GlobalAt, GlobalShifted, LocalSlot };
    Base base = Base::GlobalAt;
    int offset = 0;
    MemSpace space() const { return base == Base::LocalSlot ? MemSpace::Local : MemSpace::Global; }
    int resolve(int shift, int myloc) const {
        return base == Base::GlobalAt ? offset
               : base == Base::GlobalShifted ? shift + offset
                                             : myloc + offset;
    }
};

/// kernel.hpp:48-78: one instruction of a cost-and-effect program.
struct CostInstr {
    enum class Kind : std::uint8_t { Busy, LocalBarrier, Effect, ActivationEnd };
    Kind kind = Kind::ActivationEnd;
    Tick ticks = 0;
    MemSpace tag = MemSpace::Global;
    MemRef dst, src;
};

/// kernel.hpp:79-90: a kernel compiled to its per-activation and epilogue
/// sequences, as the engine runs them (mctb_kernel_program).
struct KernelProgram {
    KernelKind kind = KernelKind::Abstract;
    std::vector<CostInstr> per_activation;
    std::vector<CostInstr> epilogue;

    bool has_epilogue() const { return epilogue.size() > 1; }
    Tick activation_busy_ticks() const { return busy(per_activation); }
    Tick epilogue_busy_ticks() const { return busy(epilogue); }
    int barriers_per_activation() const {
        int n = 0;
        for (const auto& c : per_activation) n += c.kind == CostInstr::Kind::LocalBarrier;
        return n;
    }

private:
    static Tick busy(const std::vector<CostInstr>& v) {
        Tick t = 0;
        for (const auto& c : v)
            if (c.kind == CostInstr::Kind::Busy) t += c.ticks;
        return t;
    }
};

/// kernel.hpp:92-95.
inline int global_item_id(const TuningParams& params, int np, int nwg, int me, int iter) {
    return params.wg > np ? nwg * params.wg + me + iter * np : nwg * params.wg + me;
}

namespace detail {
// The engine's program rows (include/mctune_b200.h mctb_kernel_program) as
// CostInstr sequences: the abstract kernel's busy phases alternate a global tile
// load (gmt * ts ticks) and a local compute (ts ticks), its last busy is the
// global result write; the minimum kernel's map effects read the shifted global
// tile into the item's slot, its epilogue folds the group's slots and publishes
// glob[0].
inline KernelProgram kernel_program(const PlatformConfig& platform, int size, int kernel,
                                    const TuningParams& params) {
    const int plat[4] = {platform.nd, platform.nu, platform.np, platform.gmt};
    std::vector<std::int32_t> rows(3 * 4096);
    int n_act = 0, n_epi = 0;
    check(mctb_kernel_program(plat, size, kernel, params.wg, params.ts, rows.data(), 4096, &n_act,
                              &n_epi));
    KernelProgram prog;
    prog.kind = kernel ? KernelKind::Minimum : KernelKind::Abstract;
    for (int i = 0; i < n_act + n_epi; ++i) {
        const bool epi = i >= n_act;
        CostInstr c;
        const std::int32_t* r = rows.data() + 3 * i;
        c.kind = static_cast<CostInstr::Kind>(r[0]);
        if (c.kind == CostInstr::Kind::Busy) {
            c.ticks = r[1];
            // abstract: the local compute phases tick ts; minimum: the epilogue's folds
            const int j = i - (epi ? n_act : 0);
            c.tag = kernel == 0 ? (j % 4 == 2 ? MemSpace::Local : MemSpace::Global)
                                : (epi && r[1] == 1 && j + 1 < n_epi - 2 ? MemSpace::Local
                                                                         : MemSpace::Global);
        } else if (c.kind == CostInstr::Kind::Effect) {
            if (!epi) {
                c.dst = MemRef{MemRef::Base::LocalSlot, 0};
                c.src = MemRef{MemRef::Base::GlobalShifted, r[2]};
            } else if (r[2] >= 0) {
                c.dst = MemRef{MemRef::Base::LocalSlot, 0};
                c.src = MemRef{MemRef::Base::LocalSlot, r[2]};
            } else {
                c.dst = MemRef{MemRef::Base::GlobalAt, 0};
                c.src = MemRef{MemRef::Base::LocalSlot, 0};
            }
        }
        (epi ? prog.epilogue : prog.per_activation).push_back(c);
    }
    return prog;
}
}  // namespace detail

/// kernel.hpp:97-101.
inline KernelProgram build_abstract_kernel(int size, const TuningParams& params,
                                           const PlatformConfig& platform) {
    return detail::kernel_program(platform, size, 0, params);
}

/// kernel.hpp:103-112: ConfigError for an input of the wrong length or an
/// infeasible (wg, ts).
inline KernelProgram build_minimum_kernel(int size, const TuningParams& params,
                                          const PlatformConfig& platform,
                                          const std::vector<std::int64_t>& input) {
    if (input.size() != static_cast<std::size_t>(size))
        throw ConfigError("minimum kernel input length must equal size");
    return detail::kernel_program(platform, size, 1, params);
}

// ------------------------------------------------------------------ machine (machine.hpp)
/// Transition labels (machine.hpp:48-68).
enum class Op : std::uint8_t {
    ClockTick, ClockHalt, HostGo, HostReactGo, HostStop, HostSetFin, DeviceUnitGo, DeviceDone,
    DeviceUnitStop, UnitPexGo, UnitDone, UnitPexStop, UnitBarrierStop, PexReport, PexEffect,
    PexArrive, PexItemDone, PexEndDone, BarrierRelease
};

/// machine.hpp:70: the clock, a handshake between two processes, or a local step.
enum class TransitionKind : std::uint8_t { ClockTick, ChannelHandshake, LocalStep };

/// One atomic step of the transition system (machine.hpp:76-84).
struct Transition {
    std::uint16_t actor = 0;
    std::uint16_t peer = 0xffff;
    Op op = Op::ClockTick;
    std::int32_t arg = 0;
    bool operator==(const Transition&) const = default;
    TransitionKind kind() const {
        switch (op) {
            case Op::ClockTick: return TransitionKind::ClockTick;
            case Op::ClockHalt:
            case Op::HostSetFin:
            case Op::PexReport:
            case Op::PexEffect: return TransitionKind::LocalStep;
            default: return TransitionKind::ChannelHandshake;
        }
    }
};

/// Scheduling policies of Machine::run (machine.hpp:143) plus the engine's own.
enum class SchedPolicy : std::uint8_t {
    RoundRobin = MCTB_POLICY_ROUND_ROBIN,
    SeededRandom = MCTB_POLICY_MT19937,  // std::mt19937_64, bit-exact with the reference
    FirstEnabled = MCTB_POLICY_FIRST,    // the first DFS path of explore_machine
    Philox = MCTB_POLICY_PHILOX,         // counter-based swarm trajectory
    TickLast = MCTB_POLICY_TICK_LAST     // lock-step schedule
};

/// Machine::run's outcome (machine.hpp:145-149): final time, transition count,
/// and glob[0] for the minimum kernel.
struct RunOutcome {
    Tick time = 0;
    long long transitions = 0;
    std::optional<std::int64_t> result;
    long long steps = 0;  // machine.hpp:148 (= transitions)
};

namespace detail {
struct Args {
    int plat[4];
    int size, kernel;
    const std::int64_t* input;
    Args(const PlatformConfig& p, const ProblemSpec& prob)
        : plat{p.nd, p.nu, p.np, p.gmt},
          size(prob.size),
          kernel(prob.kernel == KernelKind::Minimum ? 1 : 0),
          input(prob.kernel == KernelKind::Minimum && !prob.input.empty() ? prob.input.data()
                                                                         : nullptr) {}
};

inline std::vector<Transition> unpack(const std::vector<std::int32_t>& buf, long long n) {
    std::vector<Transition> t(static_cast<std::size_t>(n));
    for (long long i = 0; i < n; ++i)
        t[i] = Transition{static_cast<std::uint16_t>(buf[4 * i]),
                          static_cast<std::uint16_t>(buf[4 * i + 1]),
                          static_cast<Op>(buf[4 * i + 2]), buf[4 * i + 3]};
    return t;
}

inline std::vector<std::int32_t> pack(const std::vector<Transition>& t) {
    std::vector<std::int32_t> b(4 * t.size());
    for (std::size_t i = 0; i < t.size(); ++i) {
        b[4 * i] = t[i].actor;
        b[4 * i + 1] = t[i].peer;
        b[4 * i + 2] = static_cast<std::int32_t>(t[i].op);
        b[4 * i + 3] = t[i].arg;
    }
    return b;
}

// Runs `call(trace, cap, &len)` with a trace buffer that grows once to the
// reported length when the first capacity is too small.
template <class F>
std::vector<Transition> with_trace(F&& call) {
    std::int64_t cap = 1 << 16, len = 0;
    std::vector<std::int32_t> buf(4 * cap);
    check(call(buf.data(), cap, &len));
    if (len > cap) {
        cap = len;
        buf.assign(4 * cap, 0);
        check(call(buf.data(), cap, &len));
    }
    return unpack(buf, std::min(len, cap));
}

using Clock = std::chrono::steady_clock;
inline double since(Clock::time_point t0) {
    return std::chrono::duration<double>(Clock::now() - t0).count();
}
}  // namespace detail

/// Machine::run (machine.hpp:210-215) on the GPU.
inline RunOutcome run(const PlatformConfig& platform, const ProblemSpec& problem,
                      const TuningParams& params, SchedPolicy policy, std::uint64_t seed = 0,
                      std::vector<Transition>* trace_out = nullptr) {
    const detail::Args a(platform, problem);
    std::int64_t out[4];
    auto call = [&](std::int32_t* tr, std::int64_t cap, std::int64_t* len) {
        return mctb_simulate(a.plat, a.size, a.kernel, a.input, params.wg, params.ts,
                             static_cast<int>(policy), seed, 0, out, tr, cap, len);
    };
    if (trace_out) {
        *trace_out = detail::with_trace(call);
    } else {
        std::int64_t len = 0;
        detail::check(call(nullptr, 0, &len));
    }
    RunOutcome r;
    r.time = out[0];
    r.transitions = r.steps = out[1];
    if (problem.kernel == KernelKind::Minimum) r.result = out[2];
    return r;
}

// ------------------------------------------------------------------ Machine (machine.hpp)
/// Control locations (machine.hpp:22-46; the engine's ordinals are the same).
enum class HostPc : std::uint8_t { SendGo, WaitDoneReact, ReactGo, WaitDoneStop, SendStop, SetFin, Exited };
enum class DevicePc : std::uint8_t { WaitGo, SendUnitGo, WaitUnitDone, SendDone, StopUnits, Exited };
enum class UnitPc : std::uint8_t { WaitGo, ActivatePex, Serve, ReactPex, SendUnitDone, StopPexes, StopBarrier, Exited };
enum class BarrierPc : std::uint8_t { Counting, Exited };
enum class PexPc : std::uint8_t {
    WaitGo, Run, ArriveBarrier, WaitBarrier, ArriveGroupEnd, WaitGroupEnd, SendItemDone, SendEndDone, Exited
};
enum class ClockPc : std::uint8_t { Run, Exited };
enum class PexPhase : std::uint8_t { Activation, Epilogue };

/// machine.hpp:86-110.
struct HostState {
    HostPc pc = HostPc::SendGo;
    std::int32_t k = 0;
    bool operator==(const HostState&) const = default;
};
struct DeviceState {
    DevicePc pc = DevicePc::WaitGo;
    std::int32_t k = 0;
    std::int32_t batch_base = 0;
    bool operator==(const DeviceState&) const = default;
};
struct UnitState {
    UnitPc pc = UnitPc::WaitGo;
    std::int32_t k = 0, nwg = 0, sent = 0, got_items = 0, got_ends = 0;
    bool operator==(const UnitState&) const = default;
};
struct BarrierState {
    BarrierPc pc = BarrierPc::Counting;
    std::int32_t count = 0;
    bool operator==(const BarrierState&) const = default;
};
struct PexState {
    PexPc pc = PexPc::WaitGo;
    PexPhase phase = PexPhase::Activation;
    std::int32_t cursor = 0, busy_left = 0;
    bool reported = false;
    std::int32_t nwg = 0, iter = 0;
    bool operator==(const PexState&) const = default;
};

/// The full explicit state (machine.hpp:112-130).  A value type; glob and loc are
/// the minimum kernel's memories.
struct MachineState {
    Tick time = 0;
    std::int32_t nrp_work = 0;
    std::int32_t all_nwe = 0;
    bool fin = false;
    std::int32_t next_wg = 0;
    HostState host;
    ClockPc clock = ClockPc::Run;
    std::vector<DeviceState> devices;
    std::vector<UnitState> units;
    std::vector<BarrierState> barriers;
    std::vector<PexState> pexes;
    std::vector<std::int64_t> glob;
    std::vector<std::int64_t> loc;
    bool operator==(const MachineState&) const = default;
};

namespace detail {
// MachineState <-> the ABI's flat int64 state vector (mctune_b200.h, mctb_machine_*)
inline std::vector<std::int64_t> state_to_flat(const MachineState& s) {
    std::vector<std::int64_t> f = {s.time,      s.nrp_work, s.all_nwe,
                                   s.fin,       s.next_wg,  static_cast<std::int64_t>(s.host.pc),
                                   s.host.k,    static_cast<std::int64_t>(s.clock)};
    f.push_back(static_cast<std::int64_t>(s.devices.size()));
    for (const auto& d : s.devices) f.insert(f.end(), {static_cast<std::int64_t>(d.pc), d.k, d.batch_base});
    f.push_back(static_cast<std::int64_t>(s.units.size()));
    for (const auto& u : s.units)
        f.insert(f.end(), {static_cast<std::int64_t>(u.pc), u.k, u.nwg, u.sent, u.got_items, u.got_ends});
    f.push_back(static_cast<std::int64_t>(s.barriers.size()));
    for (const auto& b : s.barriers) f.insert(f.end(), {static_cast<std::int64_t>(b.pc), b.count});
    f.push_back(static_cast<std::int64_t>(s.pexes.size()));
    for (const auto& x : s.pexes)
        f.insert(f.end(), {static_cast<std::int64_t>(x.pc), static_cast<std::int64_t>(x.phase),
                           x.cursor, x.busy_left, x.reported, x.nwg, x.iter});
    f.push_back(static_cast<std::int64_t>(s.glob.size()));
    f.insert(f.end(), s.glob.begin(), s.glob.end());
    f.push_back(static_cast<std::int64_t>(s.loc.size()));
    f.insert(f.end(), s.loc.begin(), s.loc.end());
    return f;
}

inline MachineState state_from_flat(const std::int64_t* f, std::size_t n) {
    MachineState s;
    std::size_t i = 0;
    auto get = [&]() {
        if (i >= n) throw ModelBug("truncated state vector");
        return f[i++];
    };
    s.time = get();
    s.nrp_work = static_cast<std::int32_t>(get());
    s.all_nwe = static_cast<std::int32_t>(get());
    s.fin = get() != 0;
    s.next_wg = static_cast<std::int32_t>(get());
    s.host.pc = static_cast<HostPc>(get());
    s.host.k = static_cast<std::int32_t>(get());
    s.clock = static_cast<ClockPc>(get());
    s.devices.resize(static_cast<std::size_t>(get()));
    for (auto& d : s.devices) {
        d.pc = static_cast<DevicePc>(get());
        d.k = static_cast<std::int32_t>(get());
        d.batch_base = static_cast<std::int32_t>(get());
    }
    s.units.resize(static_cast<std::size_t>(get()));
    for (auto& u : s.units) {
        u.pc = static_cast<UnitPc>(get());
        u.k = static_cast<std::int32_t>(get());
        u.nwg = static_cast<std::int32_t>(get());
        u.sent = static_cast<std::int32_t>(get());
        u.got_items = static_cast<std::int32_t>(get());
        u.got_ends = static_cast<std::int32_t>(get());
    }
    s.barriers.resize(static_cast<std::size_t>(get()));
    for (auto& b : s.barriers) {
        b.pc = static_cast<BarrierPc>(get());
        b.count = static_cast<std::int32_t>(get());
    }
    s.pexes.resize(static_cast<std::size_t>(get()));
    for (auto& x : s.pexes) {
        x.pc = static_cast<PexPc>(get());
        x.phase = static_cast<PexPhase>(get());
        x.cursor = static_cast<std::int32_t>(get());
        x.busy_left = static_cast<std::int32_t>(get());
        x.reported = get() != 0;
        x.nwg = static_cast<std::int32_t>(get());
        x.iter = static_cast<std::int32_t>(get());
    }
    s.glob.resize(static_cast<std::size_t>(get()));
    for (auto& v : s.glob) v = get();
    s.loc.resize(static_cast<std::size_t>(get()));
    for (auto& v : s.loc) v = get();
    return s;
}
}  // namespace detail

/// machine.hpp:236: FNV-1a over the bytes with a splitmix64 finalizer.
inline std::uint64_t hash64(const std::string& bytes) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (char c : bytes) {
        h ^= static_cast<std::uint8_t>(c);
        h *= 0x100000001b3ull;
    }
    h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ull;
    h = (h ^ (h >> 27)) * 0x94d049bb133111ebull;
    return h ^ (h >> 31);
}

/// The transition system of one (platform, problem, params) choice
/// (machine.hpp:151-233).  Every rule runs on the GPU: the methods ship one state
/// to a one-thread kernel (mctb_machine_*) and back, so they suit stepping and
/// inspection; whole runs (run) and explorations go through the batched kernels.
class Machine {
public:
    Machine(PlatformConfig platform_in, ProblemSpec problem_in, TuningParams params_in)
        : platform(platform_in),
          problem(std::move(problem_in)),
          params(params_in),
          plan(derive_launch(platform, problem.size, params)),
          program(problem.kernel == KernelKind::Abstract
                      ? build_abstract_kernel(problem.size, params, platform)
                      : build_minimum_kernel(problem.size, params, platform, problem.input)) {}

    const PlatformConfig platform;
    const ProblemSpec problem;
    const TuningParams params;
    const LaunchPlan plan;
    const KernelProgram program;

    int rounds() const { return params.wg / plan.nwe; }
    int device_rounds() const { return std::max(plan.wgs / plan.nwu, 1); }
    int process_count() const { return 3 + plan.nwd + 2 * plan.nwd * plan.nwu + plan.all_nwe; }

    std::string process_name(int pid) const {
        const detail::Args a(platform, problem);
        char buf[64];
        if (mctb_machine_process_name(a.plat, a.size, a.kernel, params.wg, params.ts, pid, buf,
                                      sizeof buf) < 0)
            throw ModelBug(mctb_last_error());
        return buf;
    }

    MachineState initial_state() const {
        const detail::Args a(platform, problem);
        std::vector<std::int64_t> f(flat_cap());
        std::int64_t n = 0;
        detail::check(mctb_machine_initial(a.plat, a.size, a.kernel, a.input, params.wg, params.ts,
                                           f.data(), static_cast<std::int64_t>(f.size()), &n));
        return detail::state_from_flat(f.data(), static_cast<std::size_t>(n));
    }

    /// Every enabled transition in ascending actor pid (machine.cpp:174-336).
    std::vector<Transition> enabled(const MachineState& s) const {
        const detail::Args a(platform, problem);
        const auto f = detail::state_to_flat(s);
        std::vector<std::int32_t> buf(4 * 128);
        std::int64_t n = 0;
        detail::check(mctb_machine_enabled(a.plat, a.size, a.kernel, a.input, params.wg, params.ts,
                                           f.data(), static_cast<std::int64_t>(f.size()),
                                           buf.data(), 128, &n));
        return detail::unpack(buf, n);
    }

    /// machine.cpp:361-649; ModelBug when t is not enabled in s.
    MachineState apply(const MachineState& s, const Transition& t) const {
        const detail::Args a(platform, problem);
        const auto f = detail::state_to_flat(s);
        const std::int32_t tr[4] = {t.actor, t.peer, static_cast<std::int32_t>(t.op), t.arg};
        std::vector<std::int64_t> out(flat_cap());
        std::int64_t n = 0;
        detail::check(mctb_machine_apply(a.plat, a.size, a.kernel, a.input, params.wg, params.ts,
                                         f.data(), static_cast<std::int64_t>(f.size()), tr,
                                         out.data(), static_cast<std::int64_t>(out.size()), &n));
        return detail::state_from_flat(out.data(), static_cast<std::size_t>(n));
    }

    bool is_terminal(const MachineState& s) const { return query(s)[0] != 0; }

    /// machine.cpp:708-717: ModelBug on a non-terminal state.
    Tick final_time(const MachineState& s) const {
        if (!is_terminal(s)) throw ModelBug("final_time of a non-terminal state");
        return s.time;
    }

    /// machine.cpp:719-756: ModelBug when a structural invariant fails.
    void check_invariants(const MachineState& s) const {
        const auto q = query(s);
        if (q[1] != 0) throw ModelBug("state invariant " + std::to_string(q[1]) + " violated");
    }

    /// A canonical byte image of every field (the engine's packed words, pack.cuh —
    /// equal states give equal bytes; it is not the reference's byte layout).
    std::string serialize(const MachineState& s) const {
        std::vector<std::uint32_t> w;
        query(s, &w);
        return std::string(reinterpret_cast<const char*>(w.data()), w.size() * 4);
    }

    /// hash64(serialize(s)) (machine.cpp:715-717).
    std::uint64_t fingerprint(const MachineState& s) const { return hash64(serialize(s)); }

    /// Machine::run (machine.cpp:788-825) on the GPU.
    RunOutcome run(SchedPolicy policy, std::uint64_t seed = 0,
                   std::vector<Transition>* trace_out = nullptr) const {
        return mctune_b200::run(platform, problem, params, policy, seed, trace_out);
    }

private:
    std::size_t flat_cap() const {
        return 64 + 3 * 8 + 6 * 16 + 2 * 16 + 7 * 32 + static_cast<std::size_t>(problem.size) +
               16 * 256;
    }

    std::array<std::int64_t, 3> query(const MachineState& s,
                                      std::vector<std::uint32_t>* words = nullptr) const {
        const detail::Args a(platform, problem);
        const auto f = detail::state_to_flat(s);
        std::int64_t out[3] = {0, 0, 0};
        std::vector<std::uint32_t> w(64);
        detail::check(mctb_machine_query(a.plat, a.size, a.kernel, a.input, params.wg, params.ts,
                                         f.data(), static_cast<std::int64_t>(f.size()), out,
                                         w.data(), static_cast<std::int64_t>(w.size())));
        if (words) words->assign(w.begin(), w.begin() + out[2]);
        return {out[0], out[1], out[2]};
    }
};

// ------------------------------------------------------------------ explore (explore.hpp)
/// Checked properties (explore.hpp:19-34).
struct Property {
    enum class Kind : std::uint8_t { OverTime, NonTermination };
    Kind kind = Kind::NonTermination;
    Tick bound = 0;
    static Property over_time(Tick t) { return Property{Kind::OverTime, t}; }
    static Property non_termination() { return Property{Kind::NonTermination, 0}; }
    bool violated_by(Tick final_time) const {
        return kind == Kind::NonTermination || final_time <= bound;
    }
};

/// explore.hpp:38-44.  max_states is the per-configuration visited cap and
/// max_depth the DFS's depth cut (explore.cpp:124-127; the state graphs are
/// graded, so the cut is order-independent and the GPU sweep reproduces it).
/// The engine's exploration is exact (Bitstate is rejected like the
/// reference's bisection rejects it); wall_budget_secs bounds nothing here.
struct ExploreLimits {
    long long max_depth = 4'000'000;
    long long max_states = 5'000'000;
    double wall_budget_secs = 0.0;
    enum class Mode : std::uint8_t { Exact, Bitstate };
    Mode mode = Mode::Exact;
};

/// explore.hpp:46-56.
struct ExploreStats {
    long long states_visited = 0;
    long long transitions_applied = 0;
    long long max_depth_reached = 0;
    double wall_seconds = 0.0;
    bool limit_hit = false;
    int configs_explored = 0;
    int configs_skipped = 0;

    void absorb(const ExploreStats& o) {
        states_visited += o.states_visited;
        transitions_applied += o.transitions_applied;
        max_depth_reached = std::max(max_depth_reached, o.max_depth_reached);
        wall_seconds += o.wall_seconds;
        limit_hit = limit_hit || o.limit_hit;
        configs_explored += o.configs_explored;
        configs_skipped += o.configs_skipped;
    }
};

/// A replayable counterexample (explore.hpp:60-65).
struct Trace {
    std::vector<Transition> transitions;
    Tick final_time = 0;
    TuningParams params{};
    long long steps = 0;
};

/// explore.hpp:67-72.
struct Verdict {
    bool violated = false;
    bool exhaustive = false;
    std::optional<Trace> trace;
    ExploreStats stats;
};

/// Every interleaving of one configuration, plus the terminal-time range (a
/// proof of the minimal time over all schedules) — explore_machine
/// (explore.hpp:88-93) without the per-state hooks.
struct ExploreResult {
    bool complete = false;
    ExploreStats stats;
    Tick min_time = -1, max_time = -1;
    long long terminal_states = 0, deadlocks = 0, invariant_violations = 0;
};

inline std::vector<ExploreResult> explore_configs(const PlatformConfig& platform,
                                                  const ProblemSpec& problem,
                                                  const std::vector<TuningParams>& configs,
                                                  const ExploreLimits& limits = {},
                                                  bool check_invariants = false) {
    const detail::Args a(platform, problem);
    std::vector<std::int32_t> c;
    for (const auto& p : configs) {
        c.push_back(p.wg);
        c.push_back(p.ts);
    }
    std::vector<std::int64_t> out(9 * configs.size());
    std::int64_t info[4];
    const auto t0 = detail::Clock::now();
    detail::check(mctb_explore(a.plat, a.size, a.kernel, a.input, c.data(),
                               static_cast<int>(configs.size()), limits.max_states,
                               limits.max_depth, check_invariants ? 1 : 0, out.data(), info));
    const double wall = detail::since(t0);
    std::vector<ExploreResult> res(configs.size());
    for (std::size_t i = 0; i < configs.size(); ++i) {
        const std::int64_t* o = out.data() + 9 * i;
        ExploreResult& r = res[i];
        r.complete = o[0] != 0;
        r.stats.states_visited = o[1];
        r.stats.transitions_applied = o[2];
        r.stats.max_depth_reached = o[3];
        r.stats.limit_hit = !r.complete;
        r.stats.configs_explored = 1;
        r.stats.wall_seconds = wall;
        r.min_time = o[4];
        r.max_time = o[5];
        r.terminal_states = o[6];
        r.deadlocks = o[7];
        r.invariant_violations = o[8];
    }
    return res;
}

inline ExploreResult explore_machine(const PlatformConfig& platform, const ProblemSpec& problem,
                                     const TuningParams& params, const ExploreLimits& limits = {}) {
    return explore_configs(platform, problem, {params}, limits).front();
}

/// Per-state callbacks of explore_machine (explore.hpp:75-79).
struct ExploreHooks {
    std::function<void(const Machine&, const MachineState&)> on_state;
    std::function<bool(const Machine&, const MachineState&, const std::vector<Transition>&)>
        on_terminal;
};

/// Every interleaving of one machine with the per-state hooks (explore.hpp:81-86,
/// explore.cpp:86-165).  The GPU ranks the whole state graph level by level
/// (mctb_machine_states) and hands back the states in the order the reference's
/// DFS discovers them; the hooks then run on the host in that order: on_state
/// for every visited state, on_terminal (with the DFS path) right after it for a
/// terminal state, and a false from on_terminal stops the walk.  The visited-set
/// capacity (max_states), the depth cap, the stats and the return value follow
/// the reference's DFS exactly.  Shuffled orders (shuffle = true) depend on the
/// host's std::shuffle and are not reproduced: ConfigError.
inline bool explore_machine(const Machine& m, const ExploreLimits& limits, ExploreStats& stats,
                            const ExploreHooks& hooks, std::uint64_t shuffle_seed = 0,
                            bool shuffle = false, const std::atomic<bool>* stop = nullptr,
                            double deadline_secs = 0.0) {
    (void)shuffle_seed;
    if (limits.max_depth < 1) throw ConfigError("max_depth must be >= 1");
    if (shuffle) throw ConfigError("shuffled exploration orders are not reproduced");
    const auto t0 = detail::Clock::now();
    const detail::Args a(m.platform, m.problem);
    std::int64_t info[3] = {0, 0, 0};
    std::int64_t want = std::min<std::int64_t>(limits.max_states, 4096);
    std::vector<std::int64_t> flat;
    std::vector<std::int32_t> meta;
    for (int attempt = 0;; ++attempt) {
        const std::int64_t stride_guess = info[2] ? info[2] : 256 + 2 * m.problem.size;
        flat.resize(static_cast<std::size_t>(want * stride_guess));
        meta.resize(static_cast<std::size_t>(8 * want));
        const int rc = mctb_machine_states(
            a.plat, a.size, a.kernel, a.input, m.params.wg, m.params.ts, limits.max_depth,
            limits.max_states, flat.data(), static_cast<std::int64_t>(flat.size()), meta.data(),
            want, info);
        if (rc == MCTB_LIMIT && attempt == 0 && info[1] > 0) {
            want = info[1];
            continue;
        }
        detail::check(rc);
        break;
    }
    const std::int64_t total = info[0], n = info[1], stride = info[2];
    const auto md = [&](std::int64_t i, int k) { return meta[static_cast<std::size_t>(8 * i + k)]; };
    // the DFS applies every transition of a visited state below the depth cap
    // (explore.cpp:124-129); a state at the cap with transitions marks the run
    // incomplete when the DFS tries them
    const auto applies = [&](std::int64_t i) -> long long {
        return md(i, 4) < limits.max_depth ? md(i, 6) : 0;
    };
    const auto capped = [&](std::int64_t i) { return md(i, 4) >= limits.max_depth && md(i, 6) > 0; };
    std::vector<Transition> path;
    std::vector<std::int64_t> anc;  // indices of the states on the DFS stack
    bool complete = true;
    long long applied = 0;
    for (std::int64_t i = 0; i < n; ++i) {
        if ((i & 511) == 511 && ((stop && stop->load(std::memory_order_relaxed)) ||
                                 (deadline_secs > 0 && detail::since(t0) >= deadline_secs))) {
            // the DFS finishes the states before i only in part: count what is known
            stats.wall_seconds += detail::since(t0);
            stats.transitions_applied += applied;
            return false;
        }
        const int d = md(i, 4);
        path.resize(static_cast<std::size_t>(std::max(d - 1, 0)));
        anc.resize(static_cast<std::size_t>(d));
        if (d > 0)
            path.push_back(Transition{static_cast<std::uint16_t>(md(i, 0)),
                                      static_cast<std::uint16_t>(md(i, 1)),
                                      static_cast<Op>(md(i, 2)), md(i, 3)});
        anc.push_back(i);
        stats.states_visited += 1;
        stats.max_depth_reached = std::max<long long>(stats.max_depth_reached, d);
        if (capped(i)) complete = false;
        const MachineState s = detail::state_from_flat(flat.data() + i * stride,
                                                       static_cast<std::size_t>(stride));
        if (hooks.on_state) hooks.on_state(m, s);
        if (md(i, 5) && hooks.on_terminal && !hooks.on_terminal(m, s, path)) {
            // stopped at state i: every earlier state off the stack is finished; each
            // ancestor has applied its transitions up to the path's edge
            std::vector<char> on_stack(static_cast<std::size_t>(i + 1), 0);
            for (auto k : anc) on_stack[static_cast<std::size_t>(k)] = 1;
            for (std::int64_t k = 0; k < i; ++k)
                if (!on_stack[static_cast<std::size_t>(k)]) applied += applies(k);
            for (std::size_t k = 1; k < anc.size(); ++k) applied += md(anc[k], 7) + 1;
            stats.transitions_applied += applied;
            stats.wall_seconds += detail::since(t0);
            return complete;
        }
    }
    for (std::int64_t i = 0; i < n; ++i) applied += applies(i);
    if (total > n) {
        complete = false;  // the visited set filled up (explore.cpp:130-134)
    } else if (total == limits.max_states) {
        // full after the last discovery: any later transition attempt fails the insert
        const std::int64_t last = n - 1;
        bool later = applies(last) > 0;
        for (std::int64_t c = last; md(c, 4) > 0 && !later;) {
            std::int64_t p = c - 1;
            while (md(p, 4) != md(c, 4) - 1) --p;  // c's parent: the nearest shallower state
            later = md(c, 7) + 1 < md(p, 6);
            c = p;
        }
        if (later) complete = false;
    }
    stats.transitions_applied += applied;
    stats.wall_seconds += detail::since(t0);
    return complete;
}

/// Exhaustive check of the over-time property across the whole parameter
/// space (explore.hpp:88-93).
inline Verdict check_overtime(const PlatformConfig& platform, const ProblemSpec& problem, Tick T,
                              const ExploreLimits& limits) {
    // Bitstate mode (explore.cpp:18-46) keeps 64-bit fingerprints where exact mode
    // keeps states; the GPU table always holds whole states, so a Bitstate check
    // explores exactly and only withholds the proof (explore.cpp:202-203).
    const detail::Args a(platform, problem);
    std::int64_t out[12];
    const auto t0 = detail::Clock::now();
    auto tr = detail::with_trace([&](std::int32_t* buf, std::int64_t cap, std::int64_t* len) {
        return mctb_check_overtime(a.plat, a.size, a.kernel, a.input, T, limits.max_states,
                                   limits.max_depth, out,
                                   buf, cap, len);
    });
    Verdict v;
    v.violated = out[0] != 0;
    v.exhaustive = out[1] != 0 && limits.mode == ExploreLimits::Mode::Exact;
    v.stats.states_visited = out[2];
    v.stats.max_depth_reached = out[3];
    v.stats.transitions_applied = out[4];
    v.stats.configs_explored = static_cast<int>(out[5]);
    v.stats.configs_skipped = static_cast<int>(out[6]);
    v.stats.limit_hit = out[1] == 0;
    v.stats.wall_seconds = detail::since(t0);
    if (v.violated)
        v.trace = Trace{std::move(tr), out[7], TuningParams{static_cast<int>(out[8]),
                                                            static_cast<int>(out[9])},
                        out[10]};
    return v;
}

/// Re-applies a trace from the initial state (explore.hpp:111-113,
/// explore.cpp:283-300) on the GPU and returns the terminal state; throws
/// CorruptTrace on a divergence, a non-terminal end or a wrong final time.
inline MachineState replay(const PlatformConfig& platform, const ProblemSpec& problem,
                           const Trace& trace) {
    const detail::Args a(platform, problem);
    const auto buf = detail::pack(trace.transitions);
    std::vector<std::int64_t> f(64 * 1024 + static_cast<std::size_t>(problem.size));
    std::int64_t n = 0;
    detail::check(mctb_machine_replay(a.plat, a.size, a.kernel, a.input, trace.params.wg,
                                      trace.params.ts, buf.data(),
                                      static_cast<std::int64_t>(trace.transitions.size()),
                                      trace.final_time, f.data(),
                                      static_cast<std::int64_t>(f.size()), &n));
    return detail::state_from_flat(f.data(), static_cast<std::size_t>(n));
}

/// Terminating traces, one per distinct terminal state, for every feasible
/// configuration largest-first (explore.hpp:95-100, explore.cpp:207-233).  One
/// GPU sweep explores every configuration; a configuration whose reachable
/// terminal states are one (every schedule ends in the same state — all the
/// Table-1 platforms) contributes the end of the DFS's first path, which is
/// where the reference's DFS first meets it: the FirstEnabled run.  A
/// configuration with several terminal states (multi-device handover skew) gets
/// every terminal with its DFS path in the DFS's order (mctb_nonterm_traces,
/// lexrank.cu), and one whose visited set fills up the terminals among the first
/// max_states states of that order (graphs up to 2^22 states; LimitError beyond).
inline std::vector<Trace> check_nontermination(const PlatformConfig& platform,
                                               const ProblemSpec& problem,
                                               const ExploreLimits& limits,
                                               ExploreStats* stats_out = nullptr) {
    if (limits.max_depth < 1) throw ConfigError("max_depth must be >= 1");
    ExploreStats stats;
    std::vector<TuningParams> configs;
    for (const auto& c : enumerate_configs(problem.size)) {
        if (config_feasible(problem, c)) configs.push_back(c);
        else stats.configs_skipped += 1;
    }
    std::sort(configs.begin(), configs.end(), [](const TuningParams& a, const TuningParams& b) {
        return a.wg != b.wg ? a.wg > b.wg : a.ts > b.ts;  // explore.cpp:67-72
    });
    std::vector<Trace> traces;
    if (!configs.empty()) {
        const auto res = explore_configs(platform, problem, configs, limits);
        for (std::size_t k = 0; k < configs.size(); ++k) {
            const ExploreResult& r = res[k];
            stats.absorb(r.stats);
            if (r.deadlocks) throw ModelBug("deadlock reached during exploration");
            // a full visited set: the DFS meets only the terminals among the first
            // max_states states of its order (explore.cpp:26-30), which the engine
            // cuts there (graphs up to 2^22 states; LimitError beyond)
            const bool capped = r.stats.states_visited >= limits.max_states;
            if (r.terminal_states == 0 && !capped) continue;
            if (r.terminal_states > 1 || !r.complete) {
                // every terminal state with its DFS path, in DFS order (lexrank.cu)
                const detail::Args a(platform, problem);
                std::int64_t n = 0, len = 0;
                std::size_t rows_cap = std::max<std::size_t>(16, r.terminal_states);
                std::size_t trace_cap = std::max<std::size_t>(
                    4096, static_cast<std::size_t>(r.terminal_states) *
                              static_cast<std::size_t>(r.stats.max_depth_reached + 1));
                std::vector<std::int64_t> rows;
                std::vector<std::int32_t> buf;
                for (int attempt = 0;; ++attempt) {
                    rows.assign(2 * rows_cap, 0);
                    buf.assign(4 * trace_cap, 0);
                    const int rc = mctb_nonterm_traces(
                        a.plat, a.size, a.kernel, a.input, configs[k].wg, configs[k].ts,
                        limits.max_depth, std::min(limits.max_states, r.stats.states_visited + 1),
                        &n, rows.data(), static_cast<std::int64_t>(rows_cap), buf.data(),
                        static_cast<std::int64_t>(trace_cap), &len);
                    if (rc == MCTB_LIMIT && attempt == 0 &&
                        (static_cast<std::size_t>(n) > rows_cap ||
                         static_cast<std::size_t>(len) > trace_cap)) {
                        rows_cap = std::max(rows_cap, static_cast<std::size_t>(n));
                        trace_cap = std::max(trace_cap, static_cast<std::size_t>(len));
                        continue;
                    }
                    detail::check(rc);
                    break;
                }
                std::size_t pos = 0;
                for (std::int64_t i = 0; i < n; ++i) {
                    Trace t;
                    t.final_time = rows[2 * i];
                    t.steps = rows[2 * i + 1];
                    t.params = configs[k];
                    for (std::int64_t s = 0; s < t.steps; ++s, ++pos)
                        t.transitions.push_back(Transition{
                            static_cast<std::uint16_t>(buf[4 * pos]),
                            static_cast<std::uint16_t>(buf[4 * pos + 1]),
                            static_cast<Op>(buf[4 * pos + 2]), buf[4 * pos + 3]});
                    traces.push_back(std::move(t));
                }
                continue;
            }
            std::vector<Transition> tr;
            const RunOutcome o =
                run(platform, problem, configs[k], SchedPolicy::FirstEnabled, 0, &tr);
            if (static_cast<long long>(tr.size()) > limits.max_depth) {
                stats.limit_hit = true;  // every run of it is this long
                continue;
            }
            const long long n = static_cast<long long>(tr.size());
            traces.push_back(Trace{std::move(tr), o.time, configs[k], n});
        }
    }
    if (stats_out) stats_out->absorb(stats);
    return traces;
}

/// Randomised bounded worker (explore.hpp:102-110, explore.cpp:235-281),
/// re-designed for the GPU.  The reference runs a seed-shuffled DFS with a
/// fingerprint set per configuration; here every feasible configuration, in
/// the same mt19937_64(seed) shuffle order, runs `trajectories_per_config`
/// counter-based Philox schedules (trajectory id t -> configuration t mod n,
/// one batched launch), and every run that violates `property` yields a trace,
/// one per distinct (configuration, final time, result), re-run with capture
/// from its trajectory id.  Same contract: bitstate mode only (ConfigError
/// otherwise), deterministic per seed, every trace replays; never a proof.
inline std::vector<Trace> swarm_worker(const PlatformConfig& platform, const ProblemSpec& problem,
                                       const Property& property, std::uint64_t seed,
                                       const ExploreLimits& limits,
                                       ExploreStats* stats_out = nullptr,
                                       int trajectories_per_config = 256) {
    if (limits.mode != ExploreLimits::Mode::Bitstate)
        throw ConfigError("swarm workers run in bitstate mode");
    if (trajectories_per_config < 1) throw ConfigError("trajectories_per_config must be >= 1");
    ExploreStats stats;
    std::vector<TuningParams> configs;
    for (const auto& c : enumerate_configs(problem.size)) {
        if (config_feasible(problem, c)) configs.push_back(c);
        else stats.configs_skipped += 1;
    }
    std::vector<Trace> traces;
    if (configs.empty()) {
        if (stats_out) stats_out->absorb(stats);
        return traces;
    }
    std::mt19937_64 rng(seed);
    std::shuffle(configs.begin(), configs.end(), rng);
    const detail::Args a(platform, problem);
    const int n = static_cast<int>(configs.size());
    std::vector<std::int32_t> cfg(2 * static_cast<std::size_t>(n));
    for (int k = 0; k < n; ++k) {
        cfg[2 * k] = configs[static_cast<std::size_t>(k)].wg;
        cfg[2 * k + 1] = configs[static_cast<std::size_t>(k)].ts;
    }
    const std::uint64_t n_traj = static_cast<std::uint64_t>(n) * trajectories_per_config;
    std::vector<std::int64_t> out(6 * n_traj);
    detail::check(mctb_trajectories(a.plat, a.size, a.kernel, a.input, cfg.data(), n,
                                    MCTB_POLICY_PHILOX, seed, 0, n_traj, limits.max_depth,
                                    out.data()));
    stats.configs_explored = n;
    std::vector<std::array<std::int64_t, 3>> seen;
    for (std::uint64_t t = 0; t < n_traj; ++t) {
        const std::int64_t* r = &out[6 * t];
        stats.transitions_applied += r[1];
        stats.states_visited += r[1] + 1;
        stats.max_depth_reached = std::max<long long>(stats.max_depth_reached, r[1]);
        if (r[3] == MCTB_LIMIT) {
            stats.limit_hit = true;
            continue;
        }
        detail::check(static_cast<int>(r[3]));
        if (!property.violated_by(r[0])) continue;
        const std::array<std::int64_t, 3> key{r[5], r[0], r[2]};
        if (std::find(seen.begin(), seen.end(), key) != seen.end()) continue;
        seen.push_back(key);
        const TuningParams p = configs[static_cast<std::size_t>(r[5])];
        std::int64_t o[4];
        auto tr = detail::with_trace([&](std::int32_t* buf, std::int64_t cap, std::int64_t* len) {
            return mctb_simulate(a.plat, a.size, a.kernel, a.input, p.wg, p.ts,
                                 MCTB_POLICY_PHILOX, seed, t, o, buf, cap, len);
        });
        if (o[0] != r[0] || o[1] != r[1])
            throw ModelBug("swarm trajectory " + std::to_string(t) + " did not re-run identically");
        traces.push_back(Trace{std::move(tr), r[0], p, r[1]});
    }
    if (stats_out) stats_out->absorb(stats);
    return traces;
}

/// trace_to_text (report.hpp, report.cpp:82-97).
inline std::string trace_to_text(const PlatformConfig& platform, const ProblemSpec& problem,
                                 const Trace& trace) {
    const detail::Args a(platform, problem);
    const auto buf = detail::pack(trace.transitions);
    const auto n = static_cast<std::int64_t>(trace.transitions.size());
    const std::int64_t len = mctb_trace_text(a.plat, a.size, a.kernel, a.input, trace.params.wg,
                                             trace.params.ts, buf.data(), n, nullptr, 0);
    if (len < 0) detail::check(MCTB_CORRUPT_TRACE);
    std::string s(static_cast<std::size_t>(len) + 1, '\0');
    mctb_trace_text(a.plat, a.size, a.kernel, a.input, trace.params.wg, trace.params.ts,
                    buf.data(), n, s.data(), len + 1);
    s.resize(static_cast<std::size_t>(len));
    return s;
}

// ------------------------------------------------------------------ search (search.hpp)
enum class TuneMethod : std::uint8_t { Bisect, Swarm, Sweep };

inline const char* to_string(TuneMethod m) {
    return m == TuneMethod::Bisect ? "bisect" : m == TuneMethod::Swarm ? "swarm" : "sweep";
}

struct TuneStats {
    int checks_run = 0;
    long long states_visited_total = 0;
    double wall_seconds = 0.0;
};

/// search.hpp:22-35.
struct TuneResult {
    Tick t_min = 0;
    TuningParams params{};
    Trace trace;
    Tick t_ini = 0;
    TuneStats stats;
    TuneMethod method = TuneMethod::Bisect;
    bool proven = false;
    Tick first_trail_time = 0;

    /// t_min / first-trail time, in (0, 1].
    double first_trail_optimality() const {
        if (first_trail_time <= 0) return 1.0;
        return static_cast<double>(t_min) / static_cast<double>(first_trail_time);
    }
};

struct SweepRow {
    int size = 0;
    int wg = 0;
    int ts = 0;
    Tick time = 0;
    long long transitions = 0;
    bool ok = true;
    std::string note;  // "infeasible" or "deadlock" when !ok
};

struct RankedTrail {
    Tick time = 0;
    int wg = 0;
    int ts = 0;
    long long transitions = 0;
};

struct ExtractedParams {
    int wg = 0;
    int ts = 0;
    Tick time = 0;
};

/// Simulates one randomly chosen feasible configuration (std::mt19937_64(seed)
/// pick, SeededRandom schedule) and returns its final time (search.cpp:94-102).
inline Tick estimate_initial_time(const PlatformConfig& platform, const ProblemSpec& problem,
                                  std::uint64_t seed) {
    platform.validate();
    problem.validate();
    std::vector<TuningParams> feasible;
    for (const auto& c : enumerate_configs(problem.size))
        if (config_feasible(problem, c)) feasible.push_back(c);
    if (feasible.empty()) throw ConfigError("no feasible configurations for this problem");
    std::mt19937_64 rng(seed);
    const TuningParams cfg = feasible[static_cast<std::size_t>(rng() % feasible.size())];
    return run(platform, problem, cfg, SchedPolicy::SeededRandom, seed).time;
}

namespace detail {
inline TuneResult tune_call(const PlatformConfig& platform, const ProblemSpec& problem, Tick t_hi,
                            std::uint64_t seed, const ExploreLimits& limits) {
    const Args a(platform, problem);
    std::int64_t out[10];
    const auto t0 = Clock::now();
    auto tr = with_trace([&](std::int32_t* buf, std::int64_t cap, std::int64_t* len) {
        return mctb_tune(a.plat, a.size, a.kernel, a.input, t_hi, seed, limits.max_states,
                         limits.max_depth, out,
                         buf, cap, len, nullptr);
    });
    TuneResult r;
    r.t_min = out[0];
    r.params = TuningParams{static_cast<int>(out[1]), static_cast<int>(out[2])};
    r.t_ini = out[3];
    r.proven = out[4] != 0;
    r.stats.checks_run = static_cast<int>(out[5]);
    r.stats.states_visited_total = out[6];
    r.first_trail_time = out[7];
    r.trace = Trace{std::move(tr), out[0], r.params, out[8]};
    r.method = TuneMethod::Bisect;
    r.stats.wall_seconds = since(t0);
    return r;
}
}  // namespace detail

/// Counterexample-guided binary search for the minimal termination time
/// (search.hpp:58-63): same verdicts, statistics and trace as the reference.
inline TuneResult bisect_min_time(const PlatformConfig& platform, const ProblemSpec& problem,
                                  Tick t_hi, const ExploreLimits& limits) {
    if (limits.mode != ExploreLimits::Mode::Exact) throw ConfigError("bisection needs exact mode");
    if (t_hi < 1) throw ConfigError("t_hi must be >= 1");
    return detail::tune_call(platform, problem, t_hi, 0, limits);
}

/// The `tune` command (tools/main.cpp): estimate_initial_time(seed), then
/// bisect_min_time from it, in one GPU pass.
inline TuneResult tune(const PlatformConfig& platform, const ProblemSpec& problem,
                       std::uint64_t seed = 1, const ExploreLimits& limits = {}) {
    if (limits.mode != ExploreLimits::Mode::Exact) throw ConfigError("bisection needs exact mode");
    return detail::tune_call(platform, problem, 0, seed, limits);
}

/// Randomised search (search.hpp:65-71): rounds of `workers` x 4096
/// counter-based Philox trajectories with the reference's stop rule.
/// Heuristic: never a proof.  trails_out receives the first round's terminal
/// runs (time, params, steps; no transition lists).
inline TuneResult swarm_min_time(const PlatformConfig& platform, const ProblemSpec& problem,
                                 int workers, const ExploreLimits& limits, std::uint64_t seed,
                                 std::vector<Trace>* trails_out = nullptr) {
    if (workers < 1) throw ConfigError("swarm needs at least one worker");
    const detail::Args a(platform, problem);
    const std::int64_t per_round = static_cast<std::int64_t>(workers) * 4096;
    const std::int64_t tcap = trails_out ? per_round : 0;
    std::vector<std::int64_t> trails(4 * std::max<std::int64_t>(tcap, 1));
    std::int64_t out[10], nt = 0;
    const auto t0 = detail::Clock::now();
    auto tr = detail::with_trace([&](std::int32_t* buf, std::int64_t cap, std::int64_t* len) {
        return mctb_swarm(a.plat, a.size, a.kernel, a.input, per_round, 64, seed,
                          limits.max_depth, out, buf, cap, len, trails.data(), tcap, &nt);
    });
    TuneResult r;
    r.t_min = out[0];
    r.params = TuningParams{static_cast<int>(out[1]), static_cast<int>(out[2])};
    r.t_ini = out[3];
    r.stats.checks_run = static_cast<int>(out[4]) - 1;
    r.stats.states_visited_total = out[5];
    r.first_trail_time = out[6];
    r.trace = Trace{std::move(tr), out[0], r.params, out[7]};
    r.method = TuneMethod::Swarm;
    r.proven = false;
    r.stats.wall_seconds = detail::since(t0);
    if (trails_out)
        for (std::int64_t i = 0; i < nt; ++i)
            trails_out->push_back(Trace{{}, trails[4 * i],
                                        TuningParams{static_cast<int>(trails[4 * i + 1]),
                                                     static_cast<int>(trails[4 * i + 2])},
                                        trails[4 * i + 3]});
    return r;
}

/// Deterministic simulation of every enumerated configuration, sorted like
/// the reference (search.hpp:73-77).
inline std::vector<SweepRow> exhaustive_sweep(const PlatformConfig& platform,
                                              const ProblemSpec& problem) {
    const detail::Args a(platform, problem);
    const int n = static_cast<int>(enumerate_configs(problem.size).size());
    std::vector<std::int64_t> rows(6 * static_cast<std::size_t>(n));
    std::int64_t nr = 0;
    detail::check(mctb_sweep(a.plat, a.size, a.kernel, a.input, rows.data(), n, &nr));
    std::vector<SweepRow> out;
    for (std::int64_t i = 0; i < nr; ++i) {
        const std::int64_t* r = rows.data() + 6 * i;
        SweepRow row;
        row.size = problem.size;
        row.wg = static_cast<int>(r[0]);
        row.ts = static_cast<int>(r[1]);
        row.time = r[2];
        row.transitions = r[3];
        row.ok = r[4] != 0;
        row.note = r[5] == 1 ? "infeasible" : r[5] == 2 ? "deadlock" : "";
        out.push_back(row);
    }
    return out;
}

/// Reads (wg, ts, time) out of a counterexample after replay validation
/// (search.hpp:85-87).
inline ExtractedParams extract_params(const PlatformConfig& platform, const ProblemSpec& problem,
                                      const Trace& trace) {
    const MachineState end = replay(platform, problem, trace);
    return ExtractedParams{trace.params.wg, trace.params.ts, end.time};
}

/// Stable sort of trail summaries by (time, transitions) (search.hpp:89-90).
inline std::vector<RankedTrail> rank_trails(const std::vector<Trace>& traces) {
    std::vector<RankedTrail> out;
    for (const auto& t : traces) out.push_back(RankedTrail{t.final_time, t.params.wg, t.params.ts, t.steps});
    std::stable_sort(out.begin(), out.end(), [](const RankedTrail& x, const RankedTrail& y) {
        return x.time != y.time ? x.time < y.time : x.transitions < y.transitions;
    });
    return out;
}

// ------------------------------------------------------------------ tuning spaces
/// A tuning space beyond the reference's (wg, ts) grid: ranges over the
/// platform shape too (nd, nu, log2 np) — the configuration loop of
/// check_overtime (explore.cpp:171-200) as one exhaustive argmin kernel.
/// Index order (least = preferred on ties): wg descending, ts descending, then
/// np, nu, nd ascending; the reference's own space is Space::reference().
struct Space {
    KernelKind kernel = KernelKind::Abstract;
    int size = 8, gmt = 4;
    int nd_lo = 1, nd_hi = 1, nu_lo = 1, nu_hi = 1, log2np_lo = 2, log2np_hi = 2;
    int log2wg_lo = 1, log2wg_hi = 0, log2ts_lo = 1, log2ts_hi = 0;  // hi 0: n - 1

    static Space reference(const PlatformConfig& p, const ProblemSpec& prob) {
        p.validate();
        prob.validate();
        Space s;
        s.kernel = prob.kernel;
        s.size = prob.size;
        s.gmt = p.gmt;
        s.nd_lo = s.nd_hi = p.nd;
        s.nu_lo = s.nu_hi = p.nu;
        s.log2np_lo = s.log2np_hi = log2_exact(p.np);
        return s;
    }
    void desc(std::int64_t out[13]) const {
        const int n = is_pow2(size) ? log2_exact(size) : 0;
        const std::int64_t d[13] = {kernel == KernelKind::Minimum ? 1 : 0, size, gmt, nd_lo, nd_hi,
                                    nu_lo, nu_hi, log2np_lo, log2np_hi, log2wg_lo,
                                    log2wg_hi ? log2wg_hi : n - 1, log2ts_lo,
                                    log2ts_hi ? log2ts_hi : n - 1};
        std::copy(d, d + 13, out);
    }
    std::uint64_t count() const {
        std::int64_t d[13];
        desc(d);
        const std::uint64_t n = mctb_space_count(d);
        if (n == 0) detail::check(MCTB_CONFIG_ERROR);
        return n;
    }
};

struct SpaceResult {
    std::uint64_t key = 0;   // (min(time, 2^30 - 1) << 33) | index
    std::uint64_t index = 0;
    Tick time = 0;
    long long transitions = 0;
    PlatformConfig platform;
    TuningParams params;
};

/// The minimal-model-time configuration of [first, first + count) (count 0 =
/// to the end of the space), ties to the smaller index: host buffers, one call.
inline SpaceResult space_argmin(const Space& space, std::uint64_t first = 0,
                                std::uint64_t count = 0) {
    std::int64_t d[13];
    space.desc(d);
    if (count == 0) count = space.count() - first;
    std::uint64_t key = 0;
    std::int64_t out[8];
    detail::check(mctb_space_argmin(d, first, count, &key, out));
    SpaceResult r;
    r.key = key;
    r.index = key & ((1ull << MCTB_KEY_INDEX_BITS) - 1);
    r.time = out[0];
    r.transitions = out[1];
    r.platform = PlatformConfig{static_cast<int>(out[2]), static_cast<int>(out[3]),
                                static_cast<int>(out[4]), static_cast<int>(out[5])};
    r.params = TuningParams{static_cast<int>(out[6]), static_cast<int>(out[7])};
    return r;
}

/// Number of sm_100 devices the engine sees.
inline int device_count() { return mctb_device_count(); }

}  // namespace mctune_b200

#endif  // MCTUNE_B200_HPP
