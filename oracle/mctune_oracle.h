/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the B200 search engine.
 *
 * A plain-C restatement of the reference mctune core
 * (/root/reference/proj/src/{model,kernel,machine,explore,search}.cpp).
 * Each function cites the reference file:line it follows.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
 * load it; the product library (paper_2305_09130_b200) never links it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * the golden vectors in tests/golden/ (generated from the reference itself by
 * tests/golden/make_golden.py via oracle/_ref) and, when oracle/_ref is built,
 * against the reference directly.
 */
#ifndef MCTUNE_ORACLE_H
#define MCTUNE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes shared with the product C-ABI */
#define MO_OK 0
#define MO_MODEL_BUG 1
#define MO_CONFIG_ERROR 2
#define MO_CORRUPT_TRACE 3
#define MO_LIMIT 4

/* scheduling policies */
#define MO_POLICY_ROUND_ROBIN 0   /* machine.cpp:809-820 */
#define MO_POLICY_MT19937 1       /* machine.cpp:807-808 (std::mt19937_64(seed)() % n) */
#define MO_POLICY_FIRST 2         /* en[0]: the first path of explore_machine's DFS */
#define MO_POLICY_PHILOX 3        /* ours: Philox4x32-10 counter-based trajectory */

typedef struct {
    int32_t actor, peer, op, arg; /* same 4 x int32 exchange format as oracle/_ref */
} mo_transition;

const char* mo_last_error(void);

/* model.cpp:72-88; out = [wgs, nwd, nwu, nwe, all_nwe] */
int mo_derive_launch(const int* plat, int size, int wg, int ts, int* out);

/* Lock-step closed form of the final time and transition count (derived from
 * the machine; pinned against the reference in tests).
 * kernel 0 abstract, 1 minimum.  out = [time, steps, feasible]. */
int mo_cost_model(const int* plat, int size, int kernel, int wg, int ts, int64_t* out);

/* Machine::run (machine.cpp:788-825) with one of the policies above.
 * out = [time, steps, result (INT64_MIN for abstract), process_count].
 * trace (optional) receives at most cap transitions; *trace_len the full count. */
int mo_simulate(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                int policy, uint64_t seed, uint64_t traj, int64_t* out, mo_transition* trace,
                int64_t cap, int64_t* trace_len);

/* Fingerprints (machine.cpp:715-717, hash64 machine.cpp:24-34) of every state along a trace */
int mo_run_fingerprints(const int* plat, int size, int kernel, const int64_t* input, int wg,
                        int ts, const mo_transition* trace, int64_t len, uint64_t* out);

/* explore_machine (explore.cpp:86-165), exact mode, one configuration.
 * out = [complete, states_visited, transitions_applied, max_depth_reached,
 *        min_final_time, max_final_time, n_terminal_states, n_distinct_times] */
int mo_explore(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
               int64_t max_depth, int64_t max_states, int64_t* out);

/* check_overtime (explore.cpp:167-205), exact mode.
 * out = [violated, exhaustive, states_visited, max_depth_reached, transitions_applied,
 *        configs_explored, configs_skipped, final_time, wg, ts, steps] */
int mo_check_overtime(const int* plat, int size, int kernel, const int64_t* input, int64_t T,
                      int64_t max_depth, int64_t max_states, int64_t* out, mo_transition* trace,
                      int64_t cap, int64_t* trace_len);

/* replay (explore.cpp:283-300).  out = [final_time, result] */
int mo_replay(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
              const mo_transition* trace, int64_t len, int64_t final_time, int64_t* out);

/* trace text (report.cpp:82-97).  Returns the full length; copies at most cap-1 bytes. */
int64_t mo_trace_text(const int* plat, int size, int kernel, const int64_t* input, int wg,
                      int ts, const mo_transition* trace, int64_t len, char* buf, int64_t cap);

/* Argmin of the cost model over a generalised tuning space (the exhaustive-evaluation
 * oracle for the GPU kernel).  Space layout in DESIGN.md §4 / include/mctune_b200.h.
 * best_time/best_index: the exact least (time, index) of the feasible configurations
 * (-1 / UINT64_MAX: none); best_key: the GPU's packed, saturating key of the range. */
int mo_space_argmin(const int64_t* space_desc, uint64_t first, uint64_t count,
                    uint64_t* best_key, int64_t* best_time, uint64_t* best_index);
int mo_space_decode(const int64_t* space_desc, uint64_t index, int* cfg /* nd,nu,np,gmt,size,kernel,wg,ts */);

/* Bulk CPU replay of trajectories (checker for mctb_trajectories) */
int mo_trajectories(const int* plat, int size, int kernel, const int64_t* input,
                    const int32_t* configs, int n_configs, int policy, uint64_t seed,
                    uint64_t traj0, uint64_t n, int64_t* out);

/* Initial state (ser == NULL) or successors of a serialized state, in the reference's
 * canonical serialization, with the reference's fingerprints (test helper). */
int64_t mo_successors(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                      const unsigned char* ser, unsigned char* out, int64_t cap, uint64_t* fps,
                      int64_t* rec_len);

/* Philox4x32-10 (Salmon et al., SC'11), counter (c0..c3), key (k0,k1) -> out[4] */
void mo_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out);

/* std::mt19937_64 first outputs for a seed (for tests) */
void mo_mt19937_64(uint64_t seed, int n, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
