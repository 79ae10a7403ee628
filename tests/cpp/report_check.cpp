// Prints the report formats (include/mctune_b200_report.hpp) for fixed inputs;
// tests/test_report.py compares them with the Python mirror (report.py) and
// reads back a config file.  Host code only: no device needed.
#include <cstdio>
#include <iostream>

#include "mctune/report.hpp"

using namespace mctune;

int main(int argc, char** argv) {
    std::vector<SweepRow> rows = {{16, 8, 2, 23, 148, true, ""}, {16, 4, 8, 0, 0, false, "infeasible"}};
    std::cout << sweep_to_csv(rows) << "@@\n" << sweep_to_json(rows) << "@@\n";
    std::cout << sweep_to_json({}) << "@@\n";
    std::vector<RankedTrail> trails = {{44, 4, 4, 1700}, {50, 2, 2, 10}};
    std::cout << trails_to_csv(8, trails) << "@@\n";
    Verdict v;
    v.violated = true;
    v.exhaustive = false;
    v.stats.states_visited = 15884;
    v.stats.max_depth_reached = 261;
    v.stats.wall_seconds = 0.0123456789;
    Trace t;
    t.final_time = 44;
    t.params = {4, 4};
    t.steps = 261;
    v.trace = t;
    std::cout << verdict_to_json(v, 44, "out/trace.txt") << "@@\n";
    Verdict h;
    h.exhaustive = true;
    std::cout << verdict_to_json(h, 43, "") << "@@\n";
    TuneResult r;
    r.t_min = 44;
    r.params = {4, 4};
    r.t_ini = 60;
    r.proven = true;
    r.first_trail_time = 48;
    r.stats.checks_run = 8;
    r.stats.states_visited_total = 15884;
    r.stats.wall_seconds = 1.0;
    r.trace.steps = 261;
    std::cout << tune_result_to_json(r, "t.txt") << "@@\n" << tune_result_to_csv(8, r) << "@@\n";
    if (argc > 1) {
        const RunConfig c = load_config_file(argv[1]);
        std::cout << c.platform.nd << ' ' << c.platform.nu << ' ' << c.platform.np << ' '
                  << c.platform.gmt << ' ' << c.problem.size << ' '
                  << (c.problem.kernel == KernelKind::Minimum ? "minimum" : "abstract");
        for (auto x : c.problem.input) std::cout << ' ' << x;
        std::cout << "\n@@\n";
    }
    if (argc > 2) {
        try {
            load_config_file(argv[2]);
            std::cout << "no error\n";
        } catch (const ConfigError& e) {
            std::cout << "ConfigError\n";
        }
    }
    return 0;
}
