/* mctune_b200 — B200-native search engine for the model-checking auto-tuner of
 * arXiv:2305.09130 ("Model Checking-based Performance Prediction and Tuning of
 * OpenCL programs").  C ABI: plain pointers and sizes only.
 *
 * Each entry point replaces one interface of the reference C++ core
 * (/root/reference/proj/include/mctune/{model,explore,search}.hpp); the citation is on the
 * declaration.  Conventions shared by all calls:
 *   plat   : int[4] = {nd, nu, np, gmt}                 (model.hpp:33-40 PlatformConfig)
 *   size   : input length, a power of two >= 4           (model.hpp:48-58 ProblemSpec)
 *   kernel : 0 = abstract, 1 = minimum                   (model.hpp:42 KernelKind)
 *   input  : int64[size] or NULL (minimum kernel; NULL = glob[i] = size - i)
 *   trace  : int32[4 * cap], one transition = {actor, peer, op, arg}
 *            (machine.hpp:76-84 Transition; op = ordinal of mctune::Op)
 *   return : MCTB_OK, or the error class of the reference exception
 *            (ConfigError -> MCTB_CONFIG_ERROR, ModelBug -> MCTB_MODEL_BUG,
 *             CorruptTrace -> MCTB_CORRUPT_TRACE); text via mctb_last_error().
 * Every compute call runs on the current CUDA device; there is no CPU path —
 * calls fail with MCTB_NO_DEVICE when no sm_100 device is present.
 */
#ifndef MCTUNE_B200_H
#define MCTUNE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCTB_OK 0
#define MCTB_MODEL_BUG 1
#define MCTB_CONFIG_ERROR 2
#define MCTB_CORRUPT_TRACE 3
#define MCTB_LIMIT 4
#define MCTB_NO_DEVICE 5
#define MCTB_CUDA_ERROR 6

/* scheduling policies for mctb_simulate (machine.hpp:143 SchedPolicy + ours) */
#define MCTB_POLICY_ROUND_ROBIN 0 /* SchedPolicy::RoundRobin */
#define MCTB_POLICY_MT19937 1     /* SchedPolicy::SeededRandom (std::mt19937_64) */
#define MCTB_POLICY_FIRST 2       /* first enabled: the first DFS path of explore_machine */
#define MCTB_POLICY_PHILOX 3      /* swarm trajectory: Philox4x32-10 counter-based choice */
#define MCTB_POLICY_TICK_LAST 4   /* clock ticks only when nothing else is enabled (lock-step) */

/* argmin key: (min(time, 2^30-1) << 33) | config index  (index < 2^33).
 * The key is exact whenever its time field is below 2^30-1.  A saturated time
 * field means every configuration of the range has time >= 2^30-1 (or is
 * infeasible); mctb_space_argmin then resolves the winner exactly with
 * mctb_space_exact_async's two passes, and so must a caller of the async call. */
#define MCTB_KEY_TIME_BITS 30
#define MCTB_KEY_INDEX_BITS 33

const char* mctb_last_error(void);
int mctb_version(void);
/* number of sm_100 devices visible (0 -> every compute call fails with MCTB_NO_DEVICE) */
int mctb_device_count(void);

/* derive_launch (model.hpp:89, model.cpp:72-88); out = {wgs, nwd, nwu, nwe, all_nwe} */
int mctb_derive_launch(const int* plat, int size, int wg, int ts, int* out);

/* ---------------------------------------------------------------------------
 * Exhaustive evaluation of a tuning space (north-star subsystem 1).
 * Space descriptor sd = int64[13]:
 *   {kernel, size, gmt, nd_lo, nd_hi, nu_lo, nu_hi,
 *    log2np_lo, log2np_hi, log2wg_lo, log2wg_hi, log2ts_lo, log2ts_hi}
 * Index order (least index = preferred on ties): wg descending, ts descending,
 * then np, nu, nd ascending — for a single platform this is exactly the
 * reference's preference "largest wg, then largest ts" (search.hpp:60-61,
 * explore.cpp:64-72).  The reference's own space for (plat, size) is
 *   {kernel, size, gmt, nd, nd, nu, nu, log2 np, log2 np, 1, n-1, 1, n-1}.
 */
uint64_t mctb_space_count(const int64_t* sd);

/* Device-resident argmin: atomically min-combines the packed key of
 * [first, first+count) into *d_key (device pointer).  No host sync, no
 * allocation; stream is a cudaStream_t (NULL = legacy default stream).
 * Replaces the config loop of check_overtime (explore.cpp:171-200). */
int mctb_space_argmin_async(const int64_t* sd, uint64_t first, uint64_t count, uint64_t* d_key,
                            void* stream);

/* Host-buffer argmin (end to end, including the host<->device copies); exact for
 * every space (a saturated key is resolved by the exact passes below).
 * out = {time, steps, nd, nu, np, gmt, wg, ts} of the winning configuration. */
int mctb_space_argmin(const int64_t* sd, uint64_t first, uint64_t count, uint64_t* key,
                      int64_t* out);

/* Exact argmin of [first, first+count) in two plain passes, no packing: *d_time =
 * the least 64-bit model time of the feasible configurations (UINT64_MAX: none),
 * then *d_index = the least index with that time (device pointers; both are reset
 * by the call).  The resolution of a saturated key (search.cpp:67-78 tie rule). */
int mctb_space_exact_async(const int64_t* sd, uint64_t first, uint64_t count, uint64_t* d_time,
                           uint64_t* d_index, void* stream);

/* Per-configuration table: d_time[i], d_steps[i] for index first+i (device
 * pointers; time = -1 for infeasible configurations). */
int mctb_space_eval_async(const int64_t* sd, uint64_t first, uint64_t count, int64_t* d_time,
                          int64_t* d_steps, void* stream);

/* Measured integer issue rate of the current device (thread operations/s over the
 * chip, the best of mctb_issue_probe's integer variants 0-2) — the roofline
 * denominator of the cost-model kernel. */
int mctb_int32_peak(double* ops_per_sec, double* ms);
/* One issue-rate probe (8 independent chains per thread, 64 warps per SM):
 * 0 IMAD + LOP3, 1 IADD3, 2 IADD3 + LOP3 + IMAD + SHF, 3 FFMA (fp32 issue). */
int mctb_issue_probe(int variant, double* ops_per_sec, double* ms);

/* ---------------------------------------------------------------------------
 * Reference-compatible drivers (host buffers).
 */

/* exhaustive_sweep (search.hpp:76, search.cpp:212-244).
 * rows = int64[6 * cap]: {wg, ts, time, transitions, ok, note(0 none, 1 infeasible, 2 deadlock)},
 * sorted exactly like the reference. */
int mctb_sweep(const int* plat, int size, int kernel, const int64_t* input, int64_t* rows,
               int64_t cap, int64_t* n_rows);

/* Machine::run (machine.hpp:210-215, machine.cpp:788-825) on the GPU, with one of the
 * MCTB_POLICY_* schedulers (traj = trajectory id for MCTB_POLICY_PHILOX).
 * out = {time, steps, result (INT64_MIN for abstract), process_count}. */
int mctb_simulate(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                  int policy, uint64_t seed, uint64_t traj, int64_t* out, int32_t* trace,
                  int64_t cap, int64_t* trace_len);

/* Batched trajectories (north-star subsystem 2; the swarm_worker runs of
 * explore.hpp:102-110 re-designed as counter-based random schedules):
 * trajectory t (= traj0 + i) runs configuration configs[t % n_configs]
 * (configs = int32[2 * n_configs] of (wg, ts)).
 * out = int64[6 * n_traj]: {time, steps, result, status, FNV-1a 64 of the trace over its
 * 32-bit words {actor, peer, op, arg} (h ^= w; h *= 0x100000001b3), config}. */
int mctb_trajectories(const int* plat, int size, int kernel, const int64_t* input,
                      const int32_t* configs, int n_configs, int policy, uint64_t seed,
                      uint64_t traj0, uint64_t n_traj, int64_t max_steps, int64_t* out);
/* Device time (CUDA events on the launching stream) of the trajectory kernel of this
 * thread's last mctb_trajectories call, in ms (the call's rate without its copies). */
double mctb_trajectories_kernel_ms(void);

/* The cost-and-effect programs of build_abstract_kernel / build_minimum_kernel
 * (kernel.hpp:92-118, kernel.cpp:26-82) as the engine runs them (host-side model
 * description, no device needed): out = int32[3 * cap] rows {kind (0 busy,
 * 1 local barrier, 2 effect, 3 end), ticks, operand}, the per-activation sequence
 * (*n_act rows) then the epilogue (*n_epi rows, 0 for the abstract kernel); an
 * effect's operand is its source offset (activation: glob[shift + operand] into
 * loc[me]; epilogue: loc[me + operand] into loc[me], or -1: loc[me] into glob[0]). */
int mctb_kernel_program(const int* plat, int size, int kernel, int wg, int ts, int32_t* out,
                        int cap, int* n_act, int* n_epi);

/* Machine introspection on one explicit state (machine.hpp:151-233), each rule in a
 * one-thread GPU kernel (capi_state.cu).  A state crosses the ABI as a flat int64
 * vector of the reference MachineState's fields (machine.hpp:112-130):
 *   {time, nrp_work, all_nwe, fin, next_wg, host_pc, host_k, clock,
 *    nwd, {pc, k, batch_base} x nwd, n_units, {pc, k, nwg, sent, got_items, got_ends} x n_units,
 *    n_units, {pc, count} x n_units, n_pex, {pc, phase, cursor, busy_left, reported, nwg, iter} x n_pex,
 *    n_glob, glob values, n_loc, loc values}   (glob/loc: minimum kernel only, else 0 entries)
 * Control locations use the ordinals of machine.hpp:22-46. */
int mctb_machine_initial(const int* plat, int size, int kernel, const int64_t* input, int wg,
                         int ts, int64_t* flat, int64_t cap, int64_t* n);
/* enabled transitions in ascending actor pid: int32[4 * cap] {actor, peer, op, arg} */
int mctb_machine_enabled(const int* plat, int size, int kernel, const int64_t* input, int wg,
                         int ts, const int64_t* flat, int64_t n, int32_t* trans, int64_t cap,
                         int64_t* n_trans);
/* apply (MCTB_MODEL_BUG when the transition t = int32[4] is not enabled) */
int mctb_machine_apply(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                       const int64_t* flat, int64_t n, const int32_t* t, int64_t* out_flat,
                       int64_t cap, int64_t* n_out);
/* out = int64[3] {is_terminal, check_invariants code (0 = holds), packed words}; words = the
 * state's canonical packed words (uint32[cap]) */
int mctb_machine_query(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                       const int64_t* flat, int64_t n, int64_t* out, uint32_t* words,
                       int64_t cap);
/* Machine::process_name (machine.cpp:103-113): the name's length, -1 on error */
int64_t mctb_machine_process_name(const int* plat, int size, int kernel, int wg, int ts, int pid,
                                  char* buf, int64_t cap);

/* replay (explore.cpp:283-300) in one GPU thread: MCTB_CORRUPT_TRACE on a divergence,
 * a non-terminal end or a final time other than final_time; the terminal state
 * (flat) goes to out_flat */
int mctb_machine_replay(const int* plat, int size, int kernel, const int64_t* input, int wg,
                        int ts, const int32_t* trace, int64_t len, int64_t final_time,
                        int64_t* out_flat, int64_t cap, int64_t* n_out);
/* explore_machine's visit order for the per-state hooks (explore.cpp:86-165): every
 * state within max_depth in the order the reference's DFS discovers it (the preorder
 * of the least-path tree, lexrank.cu), truncated to the first max_states.  flat = the
 * states (stride info[2]); meta = int32[8 * meta_cap] {in-transition actor, peer, op,
 * arg (-1 at the root), depth, terminal, enabled count, in-edge index}; info =
 * int64[3] {states in the full exploration, states returned, stride}.  MCTB_LIMIT
 * (info filled) when a buffer is too small. */
int mctb_machine_states(const int* plat, int size, int kernel, const int64_t* input, int wg,
                        int ts, int64_t max_depth, int64_t max_states, int64_t* flat,
                        int64_t flat_cap, int32_t* meta, int64_t meta_cap, int64_t* info);

/* replay (explore.hpp:111-113, explore.cpp:283-300) on the GPU; out = {final_time, result} */
int mctb_replay(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                const int32_t* trace, int64_t len, int64_t final_time, int64_t* out);

/* trace_to_text (report.hpp:33-38, report.cpp:82-97): returns the text length and
 * copies at most cap-1 bytes + NUL into buf; -1 on error. */
int64_t mctb_trace_text(const int* plat, int size, int kernel, const int64_t* input, int wg,
                        int ts, const int32_t* trace, int64_t len, char* buf, int64_t cap);

/* ---------------------------------------------------------------------------
 * Interleaving exploration and the bound-lowering driver (subsystems 3 and 4).
 */

/* explore_machine (explore.hpp:81-86) over several configurations in one GPU sweep
 * (configs = int32[2 * n] of (wg, ts)); max_states = the reference's per-machine visited
 * cap (ExploreLimits::max_states, default 5e6 when <= 0); max_depth =
 * ExploreLimits::max_depth (>= 1, else MCTB_CONFIG_ERROR as explore.cpp:91; the
 * reference default is 4e6): states deeper than it are not explored
 * (explore.cpp:124-127) and complete is 0 when one was cut; flags bit 0 = check
 * Machine::check_invariants (machine.cpp:719-756) and tick gating on every state;
 * bits 8-11 = P > 1 splits the visited set into P hash partitions on this device,
 * the exchange of the multi-GPU sweep (mctb_explore_mp_*) run on one GPU; bit 1 =
 * use the multi-GPU kernel's system-scope memory operations.
 * out = int64[9 * n]: {complete, states_visited, transitions_applied, max_depth_reached,
 *                      min_final_time, max_final_time, terminal_states, deadlocks,
 *                      invariant_violations}
 * info = int64[4]: {table slots, total states, packed key words, kernel microseconds} */
int mctb_explore(const int* plat, int size, int kernel, const int64_t* input,
                 const int32_t* configs, int n_configs, int64_t max_states, int64_t max_depth,
                 int flags, int64_t* out, int64_t* info);

/* Multi-GPU explore_machine: one process per GPU (rank r of world <= 8), each
 * owning the hash partition r of the visited set; successors owned by another
 * rank are probed, claimed and queued in that rank's table over peer memory
 * (NVLink P2P through CUDA IPC handles).  Protocol, every rank:
 *   open (exports this rank's 64-byte IPC handle) -> all-gather the handles ->
 *   connect -> barrier -> rank 0 only: seed -> barrier -> run -> barrier -> close.
 * run's out = int64[8 * n]: this rank's share per configuration {states discovered,
 * transitions applied, terminal states, min_final_time (INT64_MAX none),
 * max_final_time (-1 none), deadlocks, invariant_violations, protocol transitions
 * (max_depth_reached = this + max final time)} — sum / min / max over ranks;
 * info = int64[4]: {total table slots, packed key words, kernel microseconds, error}.
 * flags bit 0 = check invariants.  max_states as mctb_explore. */
int mctb_explore_mp_open(const int* plat, int size, int kernel, const int64_t* input,
                         const int32_t* configs, int n_configs, int64_t max_states, int world,
                         int rank, int flags, void** ctx, void* handle);
int mctb_explore_mp_connect(void* ctx, const void* handles);
int mctb_explore_mp_seed(void* ctx);
int mctb_explore_mp_run(void* ctx, int64_t* out, int64_t* info);
void mctb_explore_mp_close(void* ctx);

/* check_nontermination's traces for ONE configuration (explore.hpp:95-100,
 * explore.cpp:207-233): one trace per distinct terminal state, in the order the
 * reference's DFS meets them, each the path that DFS followed to it (lexrank.cu:
 * level-synchronous ranking of least paths).  rows = int64[2 * rows_cap]
 * {final_time, steps}; trace = the traces' transitions concatenated (int32[4 *
 * trace_cap]); *n_traces / *trace_len get the full sizes (MCTB_LIMIT when a
 * buffer is too small, or when the exploration exceeds max_states: the
 * reference's visited set then truncates in traversal order). */
int mctb_nonterm_traces(const int* plat, int size, int kernel, const int64_t* input, int wg,
                        int ts, int64_t max_depth, int64_t max_states, int64_t* n_traces,
                        int64_t* rows, int64_t rows_cap, int32_t* trace, int64_t trace_cap,
                        int64_t* trace_len);

/* check_overtime (explore.hpp:88-93), exact mode, within ExploreLimits' max_states and
 * max_depth (>= 1; the DFS meets no state deeper than max_depth, explore.cpp:124-127).
 * out = int64[12]: {violated, exhaustive, states_visited, max_depth_reached,
 *                   transitions_applied, configs_explored, configs_skipped, final_time, wg,
 *                   ts, steps, trace_exact}; the counterexample goes to trace. */
int mctb_check_overtime(const int* plat, int size, int kernel, const int64_t* input, int64_t T,
                        int64_t max_states, int64_t max_depth, int64_t* out, int32_t* trace,
                        int64_t cap, int64_t* trace_len);

/* The `tune` flow: estimate_initial_time (search.hpp:53-56) when t_hi <= 0, then
 * bisect_min_time (search.hpp:58-63); every probe within max_states / max_depth.
 * out = int64[10]: {t_min, wg, ts, t_ini, proven, checks_run, states_visited_total,
 *                   first_trail_time, steps, trace_exact}
 * info = double[5] (optional): {ms cost model, ms first paths, ms exploration,
 *                               explored states, ms exploration kernel} */
int mctb_tune(const int* plat, int size, int kernel, const int64_t* input, int64_t t_hi,
              uint64_t seed, int64_t max_states, int64_t max_depth, int64_t* out, int32_t* trace,
              int64_t cap, int64_t* trace_len, double* info);

/* The bound-lowering probes of the last mctb_tune on the calling thread, in
 * order: rows = int64[8 * cap] {T, violated, exhaustive, states_visited, wg, ts,
 * final_time, steps} (the counterexample check_overtime(T) returns for a violated
 * bound — its full trace is mctb_check_overtime(T)).  Returns the probe count. */
int64_t mctb_tune_probes(int64_t* rows, int64_t cap);

/* swarm_min_time (search.hpp:65-71) re-designed as rounds of per_round Philox
 * trajectories over every feasible configuration (max_rounds bounds the rounds).
 * out = int64[10]: {t_min, wg, ts, t_ini, rounds, transitions_total, first_trail_time,
 *                   steps, best_trajectory_id, trajectories_run}
 * trails (optional) = int64[4 * trails_cap] {time, wg, ts, steps} of round 0. */
int mctb_swarm(const int* plat, int size, int kernel, const int64_t* input, int64_t per_round,
               int max_rounds, uint64_t seed, int64_t max_steps, int64_t* out, int32_t* trace,
               int64_t cap, int64_t* trace_len, int64_t* trails, int64_t trails_cap,
               int64_t* n_trails);

#ifdef __cplusplus
}
#endif
#endif
