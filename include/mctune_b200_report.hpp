// Data formats either side of the tuning path, for C++ callers: the reference's
// <mctune/report.hpp> (report.hpp:12-47, report.cpp:13-180) — the run
// configuration file, input arrays, and the CSV/JSON tables and summaries the
// `tune`/`sweep`/`check` commands write.  Pure host formatting and parsing;
// every number in them comes from the GPU engine (mctune_b200.hpp).
//
// JSON is written the way the reference's nlohmann::json::dump(2) writes it:
// object keys sorted, two-space indent, shortest round-trip doubles with a
// ".0" on integral values.  The config reader accepts the same documents
// (a small recursive-descent parser; no third-party JSON library).
#pragma once

#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "mctune_b200.hpp"

namespace mctune_b200 {

/// Everything a command needs to run (report.hpp:12-20).
struct RunConfig {
    PlatformConfig platform;
    ProblemSpec problem = ProblemSpec::abstract(8);
    ExploreLimits limits;
    int workers = 4;
    std::uint64_t seed = 1;
    std::string output_dir = "out";
};

namespace json_detail {

// A JSON value: null, bool, number (kept as int64 when integral), string, array, object.
struct Value {
    enum class Kind { Null, Bool, Int, Real, String, Array, Object } kind = Kind::Null;
    bool b = false;
    std::int64_t i = 0;
    double d = 0.0;
    std::string s;
    std::vector<Value> a;
    std::map<std::string, Value> o;
};

struct Parser {
    const std::string& t;
    std::size_t p = 0;
    explicit Parser(const std::string& text) : t(text) {}
    [[noreturn]] void fail(const std::string& what) const {
        throw std::runtime_error(what + " at offset " + std::to_string(p));
    }
    void ws() {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
    }
    bool eat(char c) {
        ws();
        if (p < t.size() && t[p] == c) {
            ++p;
            return true;
        }
        return false;
    }
    std::string str() {
        if (!eat('"')) fail("expected a string");
        std::string out;
        while (p < t.size() && t[p] != '"') {
            char c = t[p++];
            if (c == '\\') {
                if (p >= t.size()) fail("bad escape");
                const char e = t[p++];
                switch (e) {
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': {
                        if (p + 4 > t.size()) fail("bad \\u escape");
                        const unsigned cp = std::stoul(t.substr(p, 4), nullptr, 16);
                        p += 4;
                        if (cp < 0x80) out += static_cast<char>(cp);
                        else if (cp < 0x800) {
                            out += static_cast<char>(0xC0 | (cp >> 6));
                            out += static_cast<char>(0x80 | (cp & 0x3F));
                        } else {
                            out += static_cast<char>(0xE0 | (cp >> 12));
                            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                            out += static_cast<char>(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: out += e; break;  // \" \\ \/
                }
            } else {
                out += c;
            }
        }
        if (p >= t.size()) fail("unterminated string");
        ++p;
        return out;
    }
    Value value() {
        ws();
        if (p >= t.size()) fail("unexpected end of input");
        Value v;
        const char c = t[p];
        if (c == '{') {
            ++p;
            v.kind = Value::Kind::Object;
            if (eat('}')) return v;
            do {
                std::string k = str();
                if (!eat(':')) fail("expected ':'");
                v.o[k] = value();
            } while (eat(','));
            if (!eat('}')) fail("expected '}'");
        } else if (c == '[') {
            ++p;
            v.kind = Value::Kind::Array;
            if (eat(']')) return v;
            do v.a.push_back(value());
            while (eat(','));
            if (!eat(']')) fail("expected ']'");
        } else if (c == '"') {
            v.kind = Value::Kind::String;
            v.s = str();
        } else if (t.compare(p, 4, "true") == 0) {
            p += 4;
            v.kind = Value::Kind::Bool;
            v.b = true;
        } else if (t.compare(p, 5, "false") == 0) {
            p += 5;
            v.kind = Value::Kind::Bool;
        } else if (t.compare(p, 4, "null") == 0) {
            p += 4;
        } else {
            const std::size_t q = p;
            bool real = false;
            if (p < t.size() && (t[p] == '-' || t[p] == '+')) ++p;
            while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '.' ||
                                    t[p] == 'e' || t[p] == 'E' || t[p] == '-' || t[p] == '+')) {
                real = real || t[p] == '.' || t[p] == 'e' || t[p] == 'E';
                ++p;
            }
            if (q == p) fail("unexpected character");
            const std::string num = t.substr(q, p - q);
            if (real) {
                v.kind = Value::Kind::Real;
                v.d = std::stod(num);
            } else {
                v.kind = Value::Kind::Int;
                v.i = std::stoll(num);
            }
        }
        return v;
    }
    Value document() {
        Value v = value();
        ws();
        if (p != t.size()) fail("trailing characters");
        return v;
    }
};

// nlohmann's number_integer_t / get<int>() semantics for the config fields
inline int as_int(const Value& v, const std::string& key) {
    if (v.kind == Value::Kind::Int) return static_cast<int>(v.i);
    if (v.kind == Value::Kind::Real) return static_cast<int>(v.d);
    throw std::runtime_error("type must be number for '" + key + "'");
}
inline std::string as_string(const Value& v, const std::string& key) {
    if (v.kind != Value::Kind::String)
        throw std::runtime_error("type must be string for '" + key + "'");
    return v.s;
}

// ---- writer: the subset of dump(2) the report functions produce
inline std::string quote(const std::string& s) {
    std::string out = "\"";
    for (const char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\t': out += "\\t"; break;
            case '\r': out += "\\r"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            default:
                if (static_cast<unsigned char>(c) < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", static_cast<unsigned char>(c));
                    out += buf;
                } else {
                    out += c;
                }
        }
    }
    return out + "\"";
}

inline std::string real(double d) {
    if (!std::isfinite(d)) return "null";
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, d);
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eE") == std::string::npos) s += ".0";
    return s;
}

// An object being written: values already rendered, keys kept sorted.
struct Obj {
    std::map<std::string, std::string> kv;
    Obj& put(const std::string& k, std::int64_t v) { kv[k] = std::to_string(v); return *this; }
    Obj& put(const std::string& k, int v) { kv[k] = std::to_string(v); return *this; }
    Obj& put(const std::string& k, bool v) { kv[k] = v ? "true" : "false"; return *this; }
    Obj& put(const std::string& k, double v) { kv[k] = real(v); return *this; }
    Obj& put(const std::string& k, const char* v) { kv[k] = quote(v); return *this; }
    Obj& put(const std::string& k, const std::string& v) { kv[k] = quote(v); return *this; }
    Obj& put(const std::string& k, const Obj& v) { kv[k] = "\x01" + v.dump(0); return *this; }
    std::string dump(int indent) const {
        if (kv.empty()) return "{}";
        const std::string pad(static_cast<std::size_t>(indent + 2), ' ');
        std::string out = "{\n";
        std::size_t n = 0;
        for (const auto& [k, v] : kv) {
            out += pad + quote(k) + ": ";
            if (!v.empty() && v[0] == '\x01') out += reindent(v.substr(1), indent + 2);
            else out += v;
            out += ++n < kv.size() ? ",\n" : "\n";
        }
        return out + std::string(static_cast<std::size_t>(indent), ' ') + "}";
    }
    // a nested object rendered at indent 0, shifted to its place
    static std::string reindent(const std::string& s, int by) {
        std::string out;
        const std::string pad(static_cast<std::size_t>(by), ' ');
        for (std::size_t i = 0; i < s.size(); ++i) {
            out += s[i];
            if (s[i] == '\n') out += pad;
        }
        return out;
    }
};

}  // namespace json_detail

/// One decimal integer per line; must hold exactly `expected` values (report.cpp:55-72).
inline std::vector<std::int64_t> read_input_file(const std::string& path, int expected) {
    std::ifstream in(path);
    if (!in) throw ConfigError("cannot open input file: " + path);
    std::vector<std::int64_t> values;
    std::string line;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        try {
            values.push_back(std::stoll(line));
        } catch (const std::exception&) {
            throw ConfigError("bad integer '" + line + "' in " + path);
        }
    }
    if (values.size() != static_cast<std::size_t>(expected))
        throw ConfigError("input file " + path + " holds " + std::to_string(values.size()) +
                          " values, expected " + std::to_string(expected));
    return values;
}

/// Platform/problem settings from a JSON config file (report.cpp:13-53):
///   { "platform": {"nd":1,"nu":1,"np":4,"gmt":4},
///     "problem":  {"size":8,"kernel":"abstract","input_path":"data.txt"} }
/// input_path is resolved relative to the config file's directory.
inline RunConfig load_config_file(const std::string& path) {
    using json_detail::Value;
    std::ifstream in(path);
    if (!in) throw ConfigError("cannot open config file: " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    Value j;
    try {
        j = json_detail::Parser(text).document();
    } catch (const std::exception& e) {
        throw ConfigError("bad config JSON in " + path + ": " + e.what());
    }
    RunConfig cfg;
    try {
        if (j.kind == Value::Kind::Object && j.o.count("platform")) {
            const Value& p = j.o.at("platform");
            auto field = [&](const char* k, int dflt) {
                return p.o.count(k) ? json_detail::as_int(p.o.at(k), k) : dflt;
            };
            cfg.platform.nd = field("nd", cfg.platform.nd);
            cfg.platform.nu = field("nu", cfg.platform.nu);
            cfg.platform.np = field("np", cfg.platform.np);
            cfg.platform.gmt = field("gmt", cfg.platform.gmt);
        }
        if (j.kind == Value::Kind::Object && j.o.count("problem")) {
            const Value& p = j.o.at("problem");
            const int size = p.o.count("size") ? json_detail::as_int(p.o.at("size"), "size") : 8;
            const KernelKind kind = kernel_kind_from_string(
                p.o.count("kernel") ? json_detail::as_string(p.o.at("kernel"), "kernel")
                                    : std::string("abstract"));
            if (kind == KernelKind::Minimum) {
                std::vector<std::int64_t> input;
                if (p.o.count("input_path")) {
                    const auto ipath =
                        std::filesystem::path(path).parent_path() /
                        json_detail::as_string(p.o.at("input_path"), "input_path");
                    input = read_input_file(ipath.string(), size);
                }
                cfg.problem = ProblemSpec::minimum(size, std::move(input));
            } else {
                cfg.problem = ProblemSpec::abstract(size);
            }
        }
    } catch (const ConfigError&) {
        throw;
    } catch (const std::exception& e) {
        throw ConfigError("bad config value in " + path + ": " + e.what());
    }
    cfg.platform.validate();
    return cfg;
}

/// report.cpp:74-80.
inline void write_text_file(const std::string& path, const std::string& content) {
    const auto dir = std::filesystem::path(path).parent_path();
    if (!dir.empty()) std::filesystem::create_directories(dir);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw ConfigError("cannot write file: " + path);
    out << content;
}

/// report.cpp:99-111: flagged rows keep their place with empty value fields.
inline std::string sweep_to_csv(const std::vector<SweepRow>& rows) {
    std::ostringstream os;
    os << "size,wg,ts,time,transitions\n";
    for (const auto& r : rows) {
        os << r.size << ',' << r.wg << ',' << r.ts << ',';
        if (r.ok) os << r.time << ',' << r.transitions;
        else os << ',';
        os << '\n';
    }
    return os.str();
}

/// report.cpp:113-129.
inline std::string sweep_to_json(const std::vector<SweepRow>& rows) {
    if (rows.empty()) return "[]\n";
    std::string out = "[\n";
    for (std::size_t i = 0; i < rows.size(); ++i) {
        const SweepRow& r = rows[i];
        json_detail::Obj o;
        o.put("size", r.size).put("wg", r.wg).put("ts", r.ts);
        if (r.ok) o.put("time", static_cast<std::int64_t>(r.time)).put("transitions", static_cast<std::int64_t>(r.transitions));
        else o.put("note", r.note);
        out += "  " + o.dump(2) + (i + 1 < rows.size() ? ",\n" : "\n");
    }
    return out + "]\n";
}

/// report.cpp:131-138.
inline std::string trails_to_csv(int size, const std::vector<RankedTrail>& trails) {
    std::ostringstream os;
    os << "size,wg,ts,time,transitions\n";
    for (const auto& t : trails)
        os << size << ',' << t.wg << ',' << t.ts << ',' << t.time << ',' << t.transitions << '\n';
    return os.str();
}

/// report.cpp:140-155.
inline std::string verdict_to_json(const Verdict& v, Tick T, const std::string& trace_path) {
    json_detail::Obj j;
    j.put("verdict", v.violated ? "violated" : "holds")
        .put("exhaustive", v.exhaustive)
        .put("T", static_cast<std::int64_t>(T))
        .put("states_visited", static_cast<std::int64_t>(v.stats.states_visited))
        .put("max_depth_reached", static_cast<std::int64_t>(v.stats.max_depth_reached))
        .put("wall_seconds", v.stats.wall_seconds);
    if (v.violated && v.trace) {
        j.put("final_time", static_cast<std::int64_t>(v.trace->final_time))
            .put("wg", v.trace->params.wg)
            .put("ts", v.trace->params.ts);
    }
    if (!trace_path.empty()) j.put("trace_path", trace_path);
    return j.dump(0) + "\n";
}

/// report.cpp:157-172.
inline std::string tune_result_to_json(const TuneResult& r, const std::string& trace_path) {
    json_detail::Obj stats;
    stats.put("checks_run", r.stats.checks_run)
        .put("states_visited_total", static_cast<std::int64_t>(r.stats.states_visited_total))
        .put("wall_seconds", r.stats.wall_seconds);
    json_detail::Obj j;
    j.put("method", to_string(r.method))
        .put("t_min", static_cast<std::int64_t>(r.t_min))
        .put("wg", r.params.wg)
        .put("ts", r.params.ts)
        .put("t_ini", static_cast<std::int64_t>(r.t_ini))
        .put("proven", r.proven)
        .put("first_trail_time", static_cast<std::int64_t>(r.first_trail_time))
        .put("first_trail_optimality", r.first_trail_optimality())
        .put("stats", stats);
    if (!trace_path.empty()) j.put("trace_path", trace_path);
    return j.dump(0) + "\n";
}

/// report.cpp:174-180: the tuning optimum as one row in the sweep CSV shape.
inline std::string tune_result_to_csv(int size, const TuneResult& r) {
    std::ostringstream os;
    os << "size,wg,ts,time,transitions\n"
       << size << ',' << r.params.wg << ',' << r.params.ts << ',' << r.t_min << ','
       << r.trace.steps << '\n';
    return os.str();
}

}  // namespace mctune_b200
