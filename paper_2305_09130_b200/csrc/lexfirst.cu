// The reference's counterexample for a schedule-dependent configuration.
//
// explore_machine (explore.cpp:86-165) with a visited set returns, for a
// bound T, the lexicographically first path (in enabled() order) from the
// initial state to a terminal state with time <= T.  When the first DFS path
// of the violating configuration is already fast enough that is simply the
// en[0] run (traj.cu, FIRST).  Otherwise (nd > 1 with host re-arming: some
// schedules tick while a finished device waits for its next batch) the path is
// found by a guided walk: at every state, take the first enabled transition
// whose successor can still finish within T.  "Can still finish within T" is
// decided by the lock-step (tick-last) completion of the successor — every
// zero-time transition before each tick — which is the minimum final time over
// all schedules from that state (pinned against the reference's exhaustive DFS
// traces in tests/test_search_gpu.py).  The walk keeps the current state on the
// device; each step evaluates the candidates in parallel, one thread each.
//
// The DFS also fully explores every earlier sibling it abandons; those
// siblings are returned (packed) so the caller can count the states and
// transitions the reference visits (one multi-source exploration).
#include <cstring>
#include <vector>

#include "bfs.cuh"
#include "common.cuh"
#include "pack.cuh"
#include "traj.cuh"

namespace mctb {

namespace {

__device__ int64_t finish_tick_last(const MachDesc& m, MState& s, int64_t max_steps) {
    Transition en[kMaxEnabled];
    for (int64_t step = 0; step < max_steps; ++step) {
        const int n = enabled(m, s, en, 2);
        if (n == 0) return is_terminal(m, s) ? s.time : INT64_MAX;
        const Transition tr = (en[0].op == OP_CLOCKTICK && n > 1) ? en[1] : en[0];
        if (!apply(m, s, tr)) return INT64_MAX;
    }
    return INT64_MAX;
}

__global__ void walk_init_kernel(MachDesc m, MState* cur) { initial_state(m, *cur); }

__global__ void walk_enabled_kernel(MachDesc m, const MState* cur, Transition* en, int* n) {
    *n = enabled(m, *cur, en);
}

// Candidate c: the final time of the lock-step completion after en[c].
__global__ void walk_candidates_kernel(MachDesc m, const MState* cur, const Transition* en, int n,
                                       int64_t max_steps, int64_t* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    MState s;
    copy_state(m, s, *cur);
    out[c] = apply(m, s, en[c]) ? finish_tick_last(m, s, max_steps) : INT64_MAX;
}

__global__ void walk_apply_kernel(MachDesc m, MState* cur, const Transition* en, int pick,
                                  int* ok) {
    *ok = apply(m, *cur, en[pick]) ? 1 : 0;
}

// Packs the successors en[0..n) of the current state (the abandoned siblings).
__global__ void walk_pack_kernel(BfsDesc d, const MState* cur, const Transition* en, int n,
                                 int words, uint32_t* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    MState s;
    copy_state(d.m, s, *cur);
    apply(d.m, s, en[c]);
    uint32_t key[kMaxWords];
    pack(d, 0, s, key);
    for (int k = 0; k < words; ++k) out[(size_t)c * words + k] = k < d.l.words ? key[k] : 0;
}

}  // namespace

// Returns MCTB_OK and fills path / final time / abandoned siblings (packed with
// `layout`), or MCTB_LIMIT when the walk exceeds max_len transitions.
int lexfirst_path(MachHost& h, int64_t T, int64_t max_len, const Layout& layout,
                  std::vector<int32_t>* path, int64_t* final_time, int64_t* sibling_applies,
                  std::vector<uint32_t>* siblings, int* n_siblings,
                  std::vector<uint32_t>* sibling_depths) {
    cudaStream_t st;
    MCTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int32_t* d_ids = nullptr;
    int rc = upload_desc(h, st, &d_ids);
    if (rc) return rc;
    const MachDesc m = h.d;
    BfsDesc bd;
    bd.m = m;
    bd.l = layout;
    const int words = layout.words;
    MState* d_cur = nullptr;
    Transition* d_en = nullptr;
    int* d_n = nullptr;
    int64_t* d_times = nullptr;
    uint32_t* d_pack = nullptr;
    MCTB_CUDA(cudaMallocAsync(&d_cur, sizeof(MState), st));
    MCTB_CUDA(cudaMallocAsync(&d_en, kMaxEnabled * sizeof(Transition), st));
    MCTB_CUDA(cudaMallocAsync(&d_n, 2 * sizeof(int), st));
    MCTB_CUDA(cudaMallocAsync(&d_times, kMaxEnabled * sizeof(int64_t), st));
    MCTB_CUDA(cudaMallocAsync(&d_pack, (size_t)kMaxEnabled * words * 4, st));
    int* h_n = nullptr;
    int64_t* h_times = nullptr;
    Transition* h_en = nullptr;
    MCTB_CUDA(cudaMallocHost(&h_n, 2 * sizeof(int)));
    MCTB_CUDA(cudaMallocHost(&h_times, kMaxEnabled * sizeof(int64_t)));
    MCTB_CUDA(cudaMallocHost(&h_en, kMaxEnabled * sizeof(Transition)));
    walk_init_kernel<<<1, 1, 0, st>>>(m, d_cur);
    path->clear();
    siblings->clear();
    *n_siblings = 0;
    if (sibling_depths) sibling_depths->clear();
    *sibling_applies = 0;
    *final_time = -1;
    rc = MCTB_OK;
    for (int64_t step = 0;; ++step) {
        walk_enabled_kernel<<<1, 1, 0, st>>>(m, d_cur, d_en, d_n);
        cudaMemcpyAsync(h_n, d_n, sizeof(int), cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(h_en, d_en, kMaxEnabled * sizeof(Transition), cudaMemcpyDeviceToHost, st);
        if ((rc = cuda_check(cudaStreamSynchronize(st), "walk"))) break;
        const int n = *h_n;
        if (n == 0) break;  // terminal (the candidates guaranteed it is within T)
        if (step >= max_len) {
            set_error("counterexample walk exceeds its length limit");
            rc = MCTB_LIMIT;
            break;
        }
        // the first enabled transition is usually right: test it alone first
        int pick = -1;
        for (int pass = 0; pass < 2 && pick < 0; ++pass) {
            const int lo = pass == 0 ? 0 : 1, cnt = pass == 0 ? 1 : n - 1;
            if (cnt <= 0) break;
            walk_candidates_kernel<<<(cnt + 31) / 32, 32, 0, st>>>(m, d_cur, d_en + lo, cnt,
                                                                   4 * max_len + 64, d_times + lo);
            cudaMemcpyAsync(h_times + lo, d_times + lo, cnt * sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st);
            if ((rc = cuda_check(cudaStreamSynchronize(st), "walk candidates"))) break;
            for (int c = lo; c < lo + cnt && pick < 0; ++c)
                if (h_times[c] <= T) pick = c;
        }
        if (rc) break;
        if (pick < 0) {
            set_error("model bug: no transition keeps the counterexample within T");
            rc = MCTB_MODEL_BUG;
            break;
        }
        if (pick > 0) {  // the DFS explores (and abandons) en[0..pick) first
            walk_pack_kernel<<<1, 32, 0, st>>>(bd, d_cur, d_en, pick, words, d_pack);
            const size_t old = siblings->size();
            siblings->resize(old + (size_t)pick * words);
            cudaMemcpyAsync(siblings->data() + old, d_pack, (size_t)pick * words * 4,
                            cudaMemcpyDeviceToHost, st);
            *n_siblings += pick;
            if (sibling_depths) sibling_depths->insert(sibling_depths->end(), pick, (uint32_t)(step + 1));
        }
        *sibling_applies += pick + 1;
        walk_apply_kernel<<<1, 1, 0, st>>>(m, d_cur, d_en, pick, d_n + 1);
        const Transition t = h_en[pick];
        path->insert(path->end(), {t.actor, t.peer, t.op, t.arg});
    }
    if (!rc) {
        int64_t tm = -1;
        cudaMemcpyAsync(&tm, &d_cur->time, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        rc = cuda_check(cudaStreamSynchronize(st), "walk time");
        *final_time = tm;
    }
    cudaFreeAsync(d_cur, st);
    cudaFreeAsync(d_en, st);
    cudaFreeAsync(d_n, st);
    cudaFreeAsync(d_times, st);
    cudaFreeAsync(d_pack, st);
    cudaFreeAsync(d_ids, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    cudaFreeHost(h_n);
    cudaFreeHost(h_times);
    cudaFreeHost(h_en);
    return rc;
}

}  // namespace mctb
