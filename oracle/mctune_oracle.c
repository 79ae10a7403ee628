/* TEST INFRASTRUCTURE ONLY — CPU oracle (checker) for the B200 search engine.
 *
 * Plain-C restatement of the reference mctune core.  Every function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
 * legs may load this library; the product never does.
 *
 * Parity: pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py through oracle/_ref) — see tests/test_oracle.py.
 */
#include "mctune_oracle.h"

#include <limits.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */

static char g_err[512];

static void set_err(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

const char* mo_last_error(void) { return g_err; }

static int is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }

static int log2i(long long v) {
    int n = 0;
    while ((1LL << n) < v) ++n;
    return n;
}

/* ------------------------------------------------------------ model-core */

typedef struct {
    int nd, nu, np, gmt;
} plat_t;

typedef struct {
    int wgs, nwd, nwu, nwe, all_nwe;
} plan_t;

/* PlatformConfig::validate, model.cpp:12-17 */
static int validate_platform(const plat_t* p) {
    if (p->nd < 1 || p->nu < 1 || p->np < 1 || p->gmt < 1) {
        set_err("platform constants nd, nu, np, gmt must all be >= 1");
        return MO_CONFIG_ERROR;
    }
    if (!is_pow2(p->np)) {
        set_err("np must be a power of two, got %d", p->np);
        return MO_CONFIG_ERROR;
    }
    return MO_OK;
}

/* validate_params, model.cpp:62-70 (+ size check of derive_launch, model.cpp:74) */
static int validate_params(int size, int wg, int ts) {
    if (size < 4 || !is_pow2(size)) {
        set_err("size must be a power of two >= 4");
        return MO_CONFIG_ERROR;
    }
    const int hi = size / 2;
    if (!is_pow2(wg) || wg < 2 || wg > hi) {
        set_err("wg must be a power of two in [2, size/2], got %d", wg);
        return MO_CONFIG_ERROR;
    }
    if (!is_pow2(ts) || ts < 2 || ts > hi) {
        set_err("ts must be a power of two in [2, size/2], got %d", ts);
        return MO_CONFIG_ERROR;
    }
    return MO_OK;
}

/* derive_launch, model.cpp:72-88: Listing 3 arithmetic, wgs clamped to >= 1 */
static void plan_of(const plat_t* p, int size, int wg, int ts, plan_t* out) {
    long long wgs = (long long)size / ((long long)wg * ts);
    if (wgs < 1) wgs = 1;
    out->wgs = (int)wgs;
    out->nwd = (out->wgs <= p->nu * p->nd) ? (out->wgs / p->nu) : p->nd;
    if (out->wgs / p->nu == 0) out->nwd = 1;
    out->nwu = (out->wgs <= p->nu) ? out->wgs : p->nu;
    out->nwe = (wg <= p->np) ? wg : p->np;
    out->all_nwe = out->nwe * out->nwu * out->nwd;
}

int mo_derive_launch(const int* plat, int size, int wg, int ts, int* out) {
    const plat_t p = {plat[0], plat[1], plat[2], plat[3]};
    int rc = validate_platform(&p);
    if (rc) return rc;
    if ((rc = validate_params(size, wg, ts))) return rc;
    plan_t pl;
    plan_of(&p, size, wg, ts, &pl);
    out[0] = pl.wgs;
    out[1] = pl.nwd;
    out[2] = pl.nwu;
    out[3] = pl.nwe;
    out[4] = pl.all_nwe;
    return MO_OK;
}

/* ---------------------------------------------------------- cost model
 * Closed form of the machine's final time and transition count under the
 * lock-step schedule.  Derivation: DESIGN.md §3.  Not a reference function —
 * it is the checker for the GPU cost-model kernel and is itself pinned against
 * Machine::run / explore_machine of the reference in tests/test_oracle.py. */
static void cost_model(const plat_t* p, int size, int kernel, int wg, int ts, int64_t* time,
                       int64_t* steps) {
    plan_t pl;
    plan_of(p, size, wg, ts, &pl);
    const int64_t rounds = wg / pl.nwe;
    int64_t dr = pl.wgs / pl.nwu; /* machine.cpp:71-72 device_rounds_ */
    if (dr < 1) dr = 1;
    const int64_t reacts = dr - pl.nwd; /* machine.cpp:73 host_reacts_ */
    const int64_t waves = (dr + pl.nwd - 1) / pl.nwd;
    const int64_t groups = dr * pl.nwu; /* workgroups actually dispatched */
    const int64_t reps = size / ts;
    const int64_t gmt = p->gmt;
    int64_t D, reports, arrivals, releases, item_done, end_done, effects;
    const int64_t items = groups * wg;
    if (kernel == 0) {
        const int64_t A = reps * (gmt * ts + ts) + gmt; /* kernel.cpp:33-43 */
        D = rounds * A;
        reports = items * A;
        arrivals = items * 2 * reps;
        releases = groups * rounds * 2 * reps;
        item_done = items;
        end_done = 0;
        effects = 0;
    } else {
        const int64_t epi = (pl.nwe - 1) + gmt; /* kernel.cpp:74-80 */
        D = rounds * ts * gmt + epi;
        reports = items * ts * gmt + groups * epi;
        arrivals = groups * pl.nwe;
        releases = groups;
        item_done = groups * (rounds - 1) * pl.nwe;
        end_done = groups * pl.nwe;
        effects = items * ts + groups * pl.nwe;
    }
    const int64_t t = waves * D;
    const int64_t host = pl.nwd + reacts + pl.nwd + 1;
    const int64_t clock = t + 1;
    const int64_t dev = dr * (pl.nwu + 1) + (int64_t)pl.nwd * pl.nwu;
    const int64_t unit = groups * (wg + 1) + (int64_t)pl.nwd * pl.nwu * (pl.nwe + 1);
    *time = t;
    *steps = host + clock + dev + unit + reports + arrivals + releases + item_done + end_done +
             effects;
}

int mo_cost_model(const int* plat, int size, int kernel, int wg, int ts, int64_t* out) {
    const plat_t p = {plat[0], plat[1], plat[2], plat[3]};
    int rc = validate_platform(&p);
    if (rc) return rc;
    if ((rc = validate_params(size, wg, ts))) return rc;
    out[2] = !(kernel == 1 && (long long)wg * ts > size); /* kernel.cpp:84-87 */
    if (!out[2]) {
        out[0] = out[1] = -1;
        return MO_OK;
    }
    cost_model(&p, size, kernel, wg, ts, &out[0], &out[1]);
    return MO_OK;
}

/* ---------------------------------------------------------------- program
 * build_abstract_kernel (kernel.cpp:26-46) / build_minimum_kernel (kernel.cpp:48-82) */

enum { IK_BUSY = 0, IK_BARRIER = 1, IK_EFFECT = 2, IK_END = 3 };
enum { MB_GLOBAL_AT = 0, MB_GLOBAL_SHIFTED = 1, MB_LOCAL_SLOT = 2 };

typedef struct {
    int kind;
    int64_t ticks;
    int dst_base, dst_off, src_base, src_off;
} instr_t;

/* ---------------------------------------------------------------- machine */

enum { R_MAIN, R_HOST, R_CLOCK, R_DEVICE, R_UNIT, R_BARRIER, R_PEX };
static const char* ROLE_NAME[] = {"main", "host", "clock", "device", "unit", "barrier", "pex"};

/* control locations, machine.hpp:22-46 (ordinals matter for serialization) */
enum { H_SENDGO, H_WAITDONEREACT, H_REACTGO, H_WAITDONESTOP, H_SENDSTOP, H_SETFIN, H_EXITED };
enum { D_WAITGO, D_SENDUNITGO, D_WAITUNITDONE, D_SENDDONE, D_STOPUNITS, D_EXITED };
enum { U_WAITGO, U_ACTIVATEPEX, U_SERVE, U_REACTPEX, U_SENDUNITDONE, U_STOPPEXES, U_STOPBARRIER,
       U_EXITED };
enum { B_COUNTING, B_EXITED };
enum { P_WAITGO, P_RUN, P_ARRIVEBARRIER, P_WAITBARRIER, P_ARRIVEGROUPEND, P_WAITGROUPEND,
       P_SENDITEMDONE, P_SENDENDDONE, P_EXITED };
enum { C_RUN, C_EXITED };
enum { PH_ACTIVATION, PH_EPILOGUE };

/* Op, machine.hpp:48-68 */
enum {
    OP_CLOCKTICK, OP_CLOCKHALT, OP_HOSTGO, OP_HOSTREACTGO, OP_HOSTSTOP, OP_HOSTSETFIN,
    OP_DEVICEUNITGO, OP_DEVICEDONE, OP_DEVICEUNITSTOP, OP_UNITPEXGO, OP_UNITDONE,
    OP_UNITPEXSTOP, OP_UNITBARRIERSTOP, OP_PEXREPORT, OP_PEXEFFECT, OP_PEXARRIVE,
    OP_PEXITEMDONE, OP_PEXENDDONE, OP_BARRIERRELEASE
};

typedef struct {
    int32_t pc, k, batch_base;
} dev_t_;
typedef struct {
    int32_t pc, k, nwg, sent, got_items, got_ends;
} unit_t_;
typedef struct {
    int32_t pc, count;
} bar_t_;
typedef struct {
    int32_t pc, phase, cursor, busy_left, reported, nwg, iter;
} pex_t_;

typedef struct {
    int64_t time;
    int32_t nrp_work, all_nwe, fin, next_wg, host_pc, host_k, clock;
    dev_t_* dev;
    unit_t_* unit;
    bar_t_* bar;
    pex_t_* pex;
    int64_t* glob;
    int64_t* loc;
} state_t;

typedef struct {
    plat_t p;
    int size, kernel, wg, ts;
    const int64_t* input;
    int64_t* default_input;
    plan_t plan;
    instr_t* act;
    int n_act;
    instr_t* epi;
    int n_epi;
    int rounds, device_rounds, host_reacts;
    int n_units, n_pex, n_glob, n_loc, n_proc;
    int* role;    /* by pid */
    int* ordinal; /* by pid */
    int* device_pid;
    int* unit_pid;
    int* barrier_pid;
    int* pex_pid;
    /* bug reporting */
    int bug;
} machine_t;

static void m_fail(machine_t* m, const char* what) {
    if (!m->bug) set_err("machine (wg=%d, ts=%d): %s", m->wg, m->ts, what);
    m->bug = 1;
}

static void machine_free(machine_t* m) {
    free(m->act);
    free(m->epi);
    free(m->role);
    free(m->ordinal);
    free(m->device_pid);
    free(m->unit_pid);
    free(m->barrier_pid);
    free(m->pex_pid);
    free(m->default_input);
    memset(m, 0, sizeof *m);
}

static void push_instr(instr_t** v, int* n, instr_t in) {
    *v = (instr_t*)realloc(*v, sizeof(instr_t) * (size_t)(*n + 1));
    (*v)[(*n)++] = in;
}

static instr_t I_busy(int64_t t) {
    instr_t i = {IK_BUSY, t, 0, 0, 0, 0};
    return i;
}
static instr_t I_barrier(void) {
    instr_t i = {IK_BARRIER, 0, 0, 0, 0, 0};
    return i;
}
static instr_t I_effect(int db, int doff, int sb, int soff) {
    instr_t i = {IK_EFFECT, 0, db, doff, sb, soff};
    return i;
}
static instr_t I_end(void) {
    instr_t i = {IK_END, 0, 0, 0, 0, 0};
    return i;
}

/* Machine::Machine, machine.cpp:60-101 */
static int machine_init(machine_t* m, const plat_t* p, int size, int kernel, const int64_t* input,
                        int wg, int ts) {
    memset(m, 0, sizeof *m);
    int rc = validate_platform(p);
    if (rc) return rc;
    if ((rc = validate_params(size, wg, ts))) return rc;
    m->p = *p;
    m->size = size;
    m->kernel = kernel;
    m->wg = wg;
    m->ts = ts;
    plan_of(p, size, wg, ts, &m->plan);
    if (kernel == 1) {
        if (!input) { /* ProblemSpec::minimum default, model.cpp:37-49 */
            m->default_input = (int64_t*)malloc(sizeof(int64_t) * (size_t)size);
            for (int i = 0; i < size; ++i) m->default_input[i] = size - i;
            input = m->default_input;
        }
        const long long top = (long long)m->plan.wgs * wg * ts; /* kernel.cpp:58-62 */
        if (top > size) {
            set_err("infeasible (wg, ts): workgroups would index past the input (%lld > %d)", top,
                    size);
            machine_free(m);
            return MO_CONFIG_ERROR;
        }
        for (int i = 0; i < ts; ++i) {
            push_instr(&m->act, &m->n_act, I_effect(MB_LOCAL_SLOT, 0, MB_GLOBAL_SHIFTED, i));
            push_instr(&m->act, &m->n_act, I_busy(p->gmt));
        }
        push_instr(&m->act, &m->n_act, I_end());
        for (int i = 1; i < m->plan.nwe; ++i) {
            push_instr(&m->epi, &m->n_epi, I_effect(MB_LOCAL_SLOT, 0, MB_LOCAL_SLOT, i));
            push_instr(&m->epi, &m->n_epi, I_busy(1));
        }
        push_instr(&m->epi, &m->n_epi, I_effect(MB_GLOBAL_AT, 0, MB_LOCAL_SLOT, 0));
        push_instr(&m->epi, &m->n_epi, I_busy(p->gmt));
        push_instr(&m->epi, &m->n_epi, I_end());
    } else {
        if (input) {
            set_err("abstract kernel takes no input array");
            return MO_CONFIG_ERROR;
        }
        const int reps = size / ts;
        for (int i = 0; i < reps; ++i) {
            push_instr(&m->act, &m->n_act, I_busy((int64_t)p->gmt * ts));
            push_instr(&m->act, &m->n_act, I_barrier());
            push_instr(&m->act, &m->n_act, I_busy(ts));
            push_instr(&m->act, &m->n_act, I_barrier());
        }
        push_instr(&m->act, &m->n_act, I_busy(p->gmt));
        push_instr(&m->act, &m->n_act, I_end());
        push_instr(&m->epi, &m->n_epi, I_end());
    }
    m->input = input;
    m->rounds = wg / m->plan.nwe;
    m->device_rounds = m->plan.wgs / m->plan.nwu;
    if (m->device_rounds < 1) m->device_rounds = 1;
    m->host_reacts = m->device_rounds - m->plan.nwd;
    m->n_units = m->plan.nwd * m->plan.nwu;
    m->n_pex = m->n_units * m->plan.nwe;
    m->n_glob = kernel == 1 ? size : 0;
    m->n_loc = kernel == 1 ? m->n_units * p->np : 0;
    m->n_proc = 3 + m->plan.nwd + 2 * m->n_units + m->n_pex;
    m->role = (int*)calloc((size_t)m->n_proc, sizeof(int));
    m->ordinal = (int*)malloc(sizeof(int) * (size_t)m->n_proc);
    for (int i = 0; i < m->n_proc; ++i) m->ordinal[i] = -1;
    m->device_pid = (int*)malloc(sizeof(int) * (size_t)m->plan.nwd);
    m->unit_pid = (int*)malloc(sizeof(int) * (size_t)m->n_units);
    m->barrier_pid = (int*)malloc(sizeof(int) * (size_t)m->n_units);
    m->pex_pid = (int*)malloc(sizeof(int) * (size_t)m->n_pex);
    int pid = 0;
    m->role[pid++] = R_MAIN;
    m->role[pid++] = R_HOST;
    m->role[pid++] = R_CLOCK;
    int g = 0, px = 0;
    for (int d = 0; d < m->plan.nwd; ++d) {
        m->device_pid[d] = pid;
        m->ordinal[pid] = d;
        m->role[pid++] = R_DEVICE;
        for (int u = 0; u < m->plan.nwu; ++u, ++g) {
            m->unit_pid[g] = pid;
            m->ordinal[pid] = g;
            m->role[pid++] = R_UNIT;
            m->barrier_pid[g] = pid;
            m->ordinal[pid] = g;
            m->role[pid++] = R_BARRIER;
            for (int e = 0; e < m->plan.nwe; ++e, ++px) {
                m->pex_pid[px] = pid;
                m->ordinal[pid] = px;
                m->role[pid++] = R_PEX;
            }
        }
    }
    return MO_OK;
}

static size_t state_bytes(const machine_t* m) {
    return sizeof(dev_t_) * (size_t)m->plan.nwd + sizeof(unit_t_) * (size_t)m->n_units +
           sizeof(bar_t_) * (size_t)m->n_units + sizeof(pex_t_) * (size_t)m->n_pex +
           sizeof(int64_t) * (size_t)(m->n_glob + m->n_loc);
}

static void state_bind(const machine_t* m, state_t* s, unsigned char* buf) {
    s->glob = (int64_t*)buf;
    buf += sizeof(int64_t) * (size_t)m->n_glob;
    s->loc = (int64_t*)buf;
    buf += sizeof(int64_t) * (size_t)m->n_loc;
    s->dev = (dev_t_*)buf;
    buf += sizeof(dev_t_) * (size_t)m->plan.nwd;
    s->unit = (unit_t_*)buf;
    buf += sizeof(unit_t_) * (size_t)m->n_units;
    s->bar = (bar_t_*)buf;
    buf += sizeof(bar_t_) * (size_t)m->n_units;
    s->pex = (pex_t_*)buf;
}

static void state_alloc(const machine_t* m, state_t* s) {
    unsigned char* buf = (unsigned char*)calloc(1, state_bytes(m) + 8);
    memset(s, 0, sizeof *s);
    state_bind(m, s, buf);
}

static void state_free(state_t* s) {
    free(s->glob);
    s->glob = NULL;
}

static void state_copy(const machine_t* m, state_t* dst, const state_t* src) {
    unsigned char* buf = (unsigned char*)dst->glob;
    memcpy(buf, src->glob, state_bytes(m));
    int64_t* g = dst->glob;
    *dst = *src;
    state_bind(m, dst, (unsigned char*)g);
}

/* Machine::initial_state, machine.cpp:115-128 */
static void initial_state(const machine_t* m, state_t* s) {
    s->time = 0;
    s->nrp_work = 0;
    s->all_nwe = m->plan.all_nwe;
    s->fin = 0;
    s->next_wg = 0;
    s->host_pc = H_SENDGO;
    s->host_k = 0;
    s->clock = C_RUN;
    memset(s->dev, 0, sizeof(dev_t_) * (size_t)m->plan.nwd);
    memset(s->unit, 0, sizeof(unit_t_) * (size_t)m->n_units);
    memset(s->bar, 0, sizeof(bar_t_) * (size_t)m->n_units);
    memset(s->pex, 0, sizeof(pex_t_) * (size_t)m->n_pex);
    for (int i = 0; i < m->n_glob; ++i) s->glob[i] = m->input[i];
    for (int i = 0; i < m->n_loc; ++i) s->loc[i] = INT64_MAX;
}

static const instr_t* instr_at(const machine_t* m, const pex_t_* px) {
    return px->phase == PH_ACTIVATION ? &m->act[px->cursor] : &m->epi[px->cursor];
}

static int has_epilogue(const machine_t* m) { return m->n_epi > 1; } /* kernel.hpp:84 */

/* Machine::place_pex, machine.cpp:136-162 */
static void place_pex(const machine_t* m, state_t* s, int p) {
    pex_t_* px = &s->pex[p];
    const instr_t* in = instr_at(m, px);
    switch (in->kind) {
        case IK_BUSY:
            px->pc = P_RUN;
            px->busy_left = (int32_t)in->ticks;
            px->reported = 0;
            break;
        case IK_EFFECT:
            px->pc = P_RUN;
            px->busy_left = 0;
            break;
        case IK_BARRIER: px->pc = P_ARRIVEBARRIER; break;
        case IK_END:
            if (px->phase == PH_EPILOGUE)
                px->pc = P_SENDENDDONE;
            else if (m->kernel == 1 && px->iter == m->rounds - 1)
                px->pc = P_ARRIVEGROUPEND;
            else
                px->pc = P_SENDITEMDONE;
            break;
    }
}

/* Machine::start_activation, machine.cpp:164-172 */
static void start_activation(const machine_t* m, state_t* s, int p, int nwg, int iter) {
    pex_t_* px = &s->pex[p];
    memset(px, 0, sizeof *px);
    px->nwg = nwg;
    px->iter = iter;
    place_pex(m, s, p);
}

typedef struct {
    mo_transition* v;
    int n, cap;
} tvec;

static void tpush(tvec* tv, int actor, int peer, int op, int arg) {
    if (tv->n == tv->cap) {
        tv->cap = tv->cap ? 2 * tv->cap : 32;
        tv->v = (mo_transition*)realloc(tv->v, sizeof(mo_transition) * (size_t)tv->cap);
    }
    mo_transition t = {actor, peer, op, arg};
    tv->v[tv->n++] = t;
}

/* Machine::enabled, machine.cpp:174-336.  The reference collects per role and
 * stable-sorts by actor pid; we emit per pid in ascending order, which yields
 * the same sequence (within one actor the emission order is unchanged). */
static void enabled(const machine_t* m, const state_t* s, tvec* out) {
    out->n = 0;
    const plan_t* pl = &m->plan;
    /* host (pid 1) */
    switch (s->host_pc) {
        case H_SENDGO:
        case H_REACTGO:
        case H_SENDSTOP: {
            const int op = s->host_pc == H_SENDGO ? OP_HOSTGO
                           : s->host_pc == H_REACTGO ? OP_HOSTREACTGO
                                                     : OP_HOSTSTOP;
            for (int d = 0; d < pl->nwd; ++d)
                if (s->dev[d].pc == D_WAITGO) tpush(out, 1, m->device_pid[d], op, s->host_k);
            break;
        }
        case H_SETFIN: tpush(out, 1, 0xffff, OP_HOSTSETFIN, 0); break;
        default: break;
    }
    /* clock (pid 2) */
    if (s->clock == C_RUN) {
        if (s->fin) tpush(out, 2, 0xffff, OP_CLOCKHALT, 0);
        if (s->all_nwe != 0 && s->nrp_work == s->all_nwe) tpush(out, 2, 0xffff, OP_CLOCKTICK, 0);
    }
    int g = 0;
    for (int d = 0; d < pl->nwd; ++d) {
        const dev_t_* dv = &s->dev[d];
        const int dpid = m->device_pid[d];
        switch (dv->pc) {
            case D_SENDUNITGO:
                for (int u = 0; u < pl->nwu; ++u)
                    if (s->unit[d * pl->nwu + u].pc == U_WAITGO)
                        tpush(out, dpid, m->unit_pid[d * pl->nwu + u], OP_DEVICEUNITGO,
                              dv->batch_base + dv->k);
                break;
            case D_SENDDONE:
                if (s->host_pc == H_WAITDONEREACT || s->host_pc == H_WAITDONESTOP)
                    tpush(out, dpid, 1, OP_DEVICEDONE, 0);
                break;
            case D_STOPUNITS:
                for (int u = 0; u < pl->nwu; ++u)
                    if (s->unit[d * pl->nwu + u].pc == U_WAITGO)
                        tpush(out, dpid, m->unit_pid[d * pl->nwu + u], OP_DEVICEUNITSTOP, 0);
                break;
            default: break;
        }
        for (int u = 0; u < pl->nwu; ++u, ++g) {
            const unit_t_* un = &s->unit[g];
            const int upid = m->unit_pid[g];
            switch (un->pc) {
                case U_ACTIVATEPEX:
                case U_REACTPEX:
                    for (int e = 0; e < pl->nwe; ++e)
                        if (s->pex[g * pl->nwe + e].pc == P_WAITGO)
                            tpush(out, upid, m->pex_pid[g * pl->nwe + e], OP_UNITPEXGO,
                                  un->sent / pl->nwe);
                    break;
                case U_SENDUNITDONE:
                    if (s->dev[d].pc == D_WAITUNITDONE)
                        tpush(out, upid, dpid, OP_UNITDONE, un->nwg);
                    break;
                case U_STOPPEXES:
                    for (int e = 0; e < pl->nwe; ++e)
                        if (s->pex[g * pl->nwe + e].pc == P_WAITGO)
                            tpush(out, upid, m->pex_pid[g * pl->nwe + e], OP_UNITPEXSTOP, 0);
                    break;
                case U_STOPBARRIER:
                    if (s->bar[g].pc == B_COUNTING && s->bar[g].count == 0)
                        tpush(out, upid, m->barrier_pid[g], OP_UNITBARRIERSTOP, 0);
                    break;
                default: break;
            }
            /* barrier */
            if (s->bar[g].pc == B_COUNTING && s->bar[g].count == pl->nwe)
                tpush(out, m->barrier_pid[g], 0xffff, OP_BARRIERRELEASE, 0);
            /* pexes */
            for (int e = 0; e < pl->nwe; ++e) {
                const int p = g * pl->nwe + e;
                const pex_t_* px = &s->pex[p];
                const int ppid = m->pex_pid[p];
                switch (px->pc) {
                    case P_RUN: {
                        const instr_t* in = instr_at(m, px);
                        if (in->kind == IK_BUSY) {
                            if (px->busy_left > 0 && !px->reported)
                                tpush(out, ppid, 0xffff, OP_PEXREPORT, 0);
                        } else if (in->kind == IK_EFFECT) {
                            tpush(out, ppid, 0xffff, OP_PEXEFFECT, px->cursor);
                        }
                        break;
                    }
                    case P_ARRIVEBARRIER:
                    case P_ARRIVEGROUPEND:
                        if (s->bar[g].pc == B_COUNTING && s->bar[g].count < pl->nwe)
                            tpush(out, ppid, m->barrier_pid[g], OP_PEXARRIVE, 0);
                        break;
                    case P_SENDITEMDONE:
                        if (un->pc == U_SERVE)
                            tpush(out, ppid, upid, OP_PEXITEMDONE, px->iter);
                        break;
                    case P_SENDENDDONE:
                        if (un->pc == U_SERVE) tpush(out, ppid, upid, OP_PEXENDDONE, 0);
                        break;
                    default: break;
                }
            }
        }
    }
}

static int pex_me(const machine_t* m, int p) { return p % m->plan.nwe; }
static int pex_unit(const machine_t* m, int p) { return p / m->plan.nwe; }

/* MemRef::resolve, kernel.hpp:28-35 + Machine::read_ref/write_ref machine.cpp:343-359 */
static int64_t* mem_ref(machine_t* m, state_t* s, int base, int off, int shift, int slot) {
    int idx;
    int64_t* arr;
    int n;
    if (base == MB_LOCAL_SLOT) {
        idx = slot + off;
        arr = s->loc;
        n = m->n_loc;
    } else {
        idx = base == MB_GLOBAL_AT ? off : shift + off;
        arr = s->glob;
        n = m->n_glob;
    }
    if (idx < 0 || idx >= n) {
        m_fail(m, "memory access out of range");
        return NULL;
    }
    return &arr[idx];
}

/* global_item_id, kernel.hpp:93-95 */
static int global_item_id(const machine_t* m, int nwg, int me, int iter) {
    return m->wg > m->p.np ? nwg * m->wg + me + iter * m->p.np : nwg * m->wg + me;
}

#define REQUIRE(c, what)          \
    do {                          \
        if (!(c)) {               \
            m_fail(m, (what));    \
            return;               \
        }                         \
    } while (0)

/* Machine::apply, machine.cpp:361-649 (in place: callers copy first) */
static void apply(machine_t* m, state_t* s, const mo_transition* t) {
    const plan_t* pl = &m->plan;
    if (t->actor < 0 || t->actor >= m->n_proc) {
        m_fail(m, "transition not enabled: bad actor");
        return;
    }
    const int peer_ok = t->peer >= 0 && t->peer < m->n_proc;
    switch (t->op) {
        case OP_CLOCKTICK: {
            REQUIRE(t->actor == 2, "transition not enabled: actor");
            REQUIRE(s->clock == C_RUN && s->all_nwe != 0 && s->nrp_work == s->all_nwe,
                    "transition not enabled: clock tick guard");
            s->nrp_work = 0;
            s->time += 1;
            for (int p = 0; p < m->n_pex; ++p) {
                pex_t_* px = &s->pex[p];
                if (!px->reported) continue;
                REQUIRE(px->pc == P_RUN && px->busy_left > 0,
                        "transition not enabled: reported element is busy");
                px->reported = 0;
                px->busy_left -= 1;
                if (px->busy_left == 0) {
                    px->cursor += 1;
                    place_pex(m, s, p);
                }
            }
            break;
        }
        case OP_CLOCKHALT:
            REQUIRE(t->actor == 2, "transition not enabled: actor");
            REQUIRE(s->clock == C_RUN && s->fin, "transition not enabled: clock halt guard");
            s->clock = C_EXITED;
            break;
        case OP_HOSTGO:
        case OP_HOSTREACTGO: {
            const int react = t->op == OP_HOSTREACTGO;
            REQUIRE(t->actor == 1, "transition not enabled: actor");
            REQUIRE(s->host_pc == (react ? H_REACTGO : H_SENDGO),
                    "transition not enabled: host send pc");
            REQUIRE(peer_ok && m->role[t->peer] == R_DEVICE, "transition not enabled: peer is a device");
            dev_t_* dv = &s->dev[m->ordinal[t->peer]];
            REQUIRE(dv->pc == D_WAITGO, "transition not enabled: device awaits go");
            if (s->next_wg + pl->nwu > pl->wgs) {
                m_fail(m, "workgroup dispatch overflow");
                return;
            }
            if (react) s->all_nwe += pl->nwe * pl->nwu;
            dv->batch_base = s->next_wg;
            s->next_wg += pl->nwu;
            dv->pc = D_SENDUNITGO;
            dv->k = 0;
            s->host_k += 1;
            if (react) {
                if (s->host_k < m->host_reacts) {
                    s->host_pc = H_WAITDONEREACT;
                } else {
                    s->host_pc = H_WAITDONESTOP;
                    s->host_k = 0;
                }
            } else if (s->host_k == pl->nwd) {
                s->host_pc = m->host_reacts > 0 ? H_WAITDONEREACT : H_WAITDONESTOP;
                s->host_k = 0;
            }
            break;
        }
        case OP_HOSTSTOP: {
            REQUIRE(t->actor == 1, "transition not enabled: actor");
            REQUIRE(s->host_pc == H_SENDSTOP, "transition not enabled: host stop pc");
            REQUIRE(peer_ok && m->role[t->peer] == R_DEVICE, "transition not enabled: peer");
            dev_t_* dv = &s->dev[m->ordinal[t->peer]];
            REQUIRE(dv->pc == D_WAITGO, "transition not enabled: device awaits stop");
            dv->pc = D_STOPUNITS;
            dv->k = 0;
            s->host_k += 1;
            s->host_pc = s->host_k == pl->nwd ? H_SETFIN : H_WAITDONESTOP;
            break;
        }
        case OP_HOSTSETFIN:
            REQUIRE(t->actor == 1, "transition not enabled: actor");
            REQUIRE(s->host_pc == H_SETFIN, "transition not enabled: host fin pc");
            s->fin = 1;
            s->host_pc = H_EXITED;
            break;
        case OP_DEVICEUNITGO: {
            REQUIRE(m->role[t->actor] == R_DEVICE, "transition not enabled: actor");
            const int d = m->ordinal[t->actor];
            dev_t_* dv = &s->dev[d];
            REQUIRE(dv->pc == D_SENDUNITGO, "transition not enabled: device go pc");
            REQUIRE(peer_ok && m->role[t->peer] == R_UNIT, "transition not enabled: peer");
            const int g = m->ordinal[t->peer];
            REQUIRE(g / pl->nwu == d, "transition not enabled: unit belongs to device");
            unit_t_* un = &s->unit[g];
            REQUIRE(un->pc == U_WAITGO, "transition not enabled: unit awaits go");
            const int nwg = dv->batch_base + dv->k;
            REQUIRE(t->arg == nwg, "transition not enabled: workgroup number matches");
            memset(un, 0, sizeof *un);
            un->pc = U_ACTIVATEPEX;
            un->nwg = nwg;
            dv->k += 1;
            if (dv->k == pl->nwu) {
                dv->pc = D_WAITUNITDONE;
                dv->k = 0;
            }
            break;
        }
        case OP_DEVICEDONE: {
            REQUIRE(m->role[t->actor] == R_DEVICE, "transition not enabled: actor");
            dev_t_* dv = &s->dev[m->ordinal[t->actor]];
            REQUIRE(dv->pc == D_SENDDONE, "transition not enabled: device done pc");
            REQUIRE(s->host_pc == H_WAITDONEREACT || s->host_pc == H_WAITDONESTOP,
                    "transition not enabled: host awaits done");
            s->host_pc = s->host_pc == H_WAITDONEREACT ? H_REACTGO : H_SENDSTOP;
            memset(dv, 0, sizeof *dv);
            break;
        }
        case OP_DEVICEUNITSTOP: {
            REQUIRE(m->role[t->actor] == R_DEVICE, "transition not enabled: actor");
            const int d = m->ordinal[t->actor];
            dev_t_* dv = &s->dev[d];
            REQUIRE(dv->pc == D_STOPUNITS, "transition not enabled: device stop pc");
            REQUIRE(peer_ok && m->role[t->peer] == R_UNIT, "transition not enabled: peer");
            const int g = m->ordinal[t->peer];
            REQUIRE(g / pl->nwu == d, "transition not enabled: unit belongs to device");
            unit_t_* un = &s->unit[g];
            REQUIRE(un->pc == U_WAITGO, "transition not enabled: unit awaits stop");
            un->pc = U_STOPPEXES;
            un->k = 0;
            dv->k += 1;
            if (dv->k == pl->nwu) dv->pc = D_EXITED;
            break;
        }
        case OP_UNITPEXGO: {
            REQUIRE(m->role[t->actor] == R_UNIT, "transition not enabled: actor");
            const int g = m->ordinal[t->actor];
            unit_t_* un = &s->unit[g];
            REQUIRE(un->pc == U_ACTIVATEPEX || un->pc == U_REACTPEX,
                    "transition not enabled: unit go pc");
            REQUIRE(peer_ok && m->role[t->peer] == R_PEX, "transition not enabled: peer");
            const int p = m->ordinal[t->peer];
            REQUIRE(pex_unit(m, p) == g, "transition not enabled: element belongs to unit");
            REQUIRE(s->pex[p].pc == P_WAITGO, "transition not enabled: element awaits go");
            const int iter = un->sent / pl->nwe;
            REQUIRE(t->arg == iter, "transition not enabled: round number matches");
            start_activation(m, s, p, un->nwg, iter);
            un->sent += 1;
            if (un->pc == U_ACTIVATEPEX) {
                un->k += 1;
                if (un->k == pl->nwe) {
                    un->pc = U_SERVE;
                    un->k = 0;
                }
            } else {
                un->pc = U_SERVE;
            }
            break;
        }
        case OP_UNITDONE: {
            REQUIRE(m->role[t->actor] == R_UNIT, "transition not enabled: actor");
            const int g = m->ordinal[t->actor];
            unit_t_* un = &s->unit[g];
            REQUIRE(un->pc == U_SENDUNITDONE, "transition not enabled: unit done pc");
            dev_t_* dv = &s->dev[g / pl->nwu];
            REQUIRE(dv->pc == D_WAITUNITDONE, "transition not enabled: device awaits unit done");
            if (m->kernel == 0) s->all_nwe -= pl->nwe;
            memset(un, 0, sizeof *un);
            dv->k += 1;
            if (dv->k == pl->nwu) {
                dv->pc = D_SENDDONE;
                dv->k = 0;
            }
            break;
        }
        case OP_UNITPEXSTOP: {
            REQUIRE(m->role[t->actor] == R_UNIT, "transition not enabled: actor");
            const int g = m->ordinal[t->actor];
            unit_t_* un = &s->unit[g];
            REQUIRE(un->pc == U_STOPPEXES, "transition not enabled: unit stop pc");
            REQUIRE(peer_ok && m->role[t->peer] == R_PEX, "transition not enabled: peer");
            const int p = m->ordinal[t->peer];
            REQUIRE(pex_unit(m, p) == g, "transition not enabled: element belongs to unit");
            REQUIRE(s->pex[p].pc == P_WAITGO, "transition not enabled: element awaits stop");
            s->pex[p].pc = P_EXITED;
            un->k += 1;
            if (un->k == pl->nwe) un->pc = U_STOPBARRIER;
            break;
        }
        case OP_UNITBARRIERSTOP: {
            REQUIRE(m->role[t->actor] == R_UNIT, "transition not enabled: actor");
            const int g = m->ordinal[t->actor];
            unit_t_* un = &s->unit[g];
            REQUIRE(un->pc == U_STOPBARRIER, "transition not enabled: unit stop-barrier pc");
            bar_t_* b = &s->bar[g];
            REQUIRE(b->pc == B_COUNTING && b->count == 0, "transition not enabled: barrier is idle");
            b->pc = B_EXITED;
            un->pc = U_EXITED;
            break;
        }
        case OP_PEXREPORT: {
            REQUIRE(m->role[t->actor] == R_PEX, "transition not enabled: actor");
            pex_t_* px = &s->pex[m->ordinal[t->actor]];
            REQUIRE(px->pc == P_RUN, "transition not enabled: element running");
            REQUIRE(instr_at(m, px)->kind == IK_BUSY && px->busy_left > 0 && !px->reported,
                    "transition not enabled: element has busy work and has not reported");
            px->reported = 1;
            s->nrp_work += 1;
            break;
        }
        case OP_PEXEFFECT: {
            REQUIRE(m->role[t->actor] == R_PEX, "transition not enabled: actor");
            const int p = m->ordinal[t->actor];
            pex_t_* px = &s->pex[p];
            REQUIRE(px->pc == P_RUN, "transition not enabled: element running");
            const instr_t* in = instr_at(m, px);
            REQUIRE(in->kind == IK_EFFECT, "transition not enabled: effect instruction");
            REQUIRE(t->arg == px->cursor, "transition not enabled: cursor matches");
            const int gid = global_item_id(m, px->nwg, pex_me(m, p), px->iter);
            const int shift = gid * m->ts;
            const int slot = pex_unit(m, p) * m->p.np + pex_me(m, p); /* machine.hpp:208 */
            const int64_t* src = mem_ref(m, s, in->src_base, in->src_off, shift, slot);
            if (!src) return;
            const int64_t v = *src;
            int64_t* dst = mem_ref(m, s, in->dst_base, in->dst_off, shift, slot);
            if (!dst) return;
            if (v < *dst) *dst = v;
            px->cursor += 1;
            place_pex(m, s, p);
            break;
        }
        case OP_PEXARRIVE: {
            REQUIRE(m->role[t->actor] == R_PEX, "transition not enabled: actor");
            const int p = m->ordinal[t->actor];
            pex_t_* px = &s->pex[p];
            REQUIRE(px->pc == P_ARRIVEBARRIER || px->pc == P_ARRIVEGROUPEND,
                    "transition not enabled: element arriving");
            bar_t_* b = &s->bar[pex_unit(m, p)];
            REQUIRE(b->pc == B_COUNTING && b->count < pl->nwe,
                    "transition not enabled: barrier counting");
            b->count += 1;
            px->pc = px->pc == P_ARRIVEBARRIER ? P_WAITBARRIER : P_WAITGROUPEND;
            break;
        }
        case OP_BARRIERRELEASE: {
            REQUIRE(m->role[t->actor] == R_BARRIER, "transition not enabled: actor");
            const int g = m->ordinal[t->actor];
            bar_t_* b = &s->bar[g];
            REQUIRE(b->pc == B_COUNTING && b->count == pl->nwe, "transition not enabled: all arrived");
            int wk = 0, wgp = 0;
            for (int e = 0; e < pl->nwe; ++e) {
                const int pc = s->pex[g * pl->nwe + e].pc;
                wk += pc == P_WAITBARRIER;
                wgp += pc == P_WAITGROUPEND;
            }
            REQUIRE(wk == pl->nwe || wgp == pl->nwe,
                    "transition not enabled: waiters at one barrier instance");
            b->count = 0;
            if (wk == pl->nwe) {
                for (int e = 0; e < pl->nwe; ++e) {
                    s->pex[g * pl->nwe + e].cursor += 1;
                    place_pex(m, s, g * pl->nwe + e);
                }
            } else {
                s->all_nwe -= pl->nwe - 1;
                for (int e = 0; e < pl->nwe; ++e) {
                    const int p = g * pl->nwe + e;
                    pex_t_* px = &s->pex[p];
                    if (pex_me(m, p) == 0 && has_epilogue(m)) {
                        px->phase = PH_EPILOGUE;
                        px->cursor = 0;
                        place_pex(m, s, p);
                    } else {
                        px->pc = P_SENDENDDONE;
                    }
                }
            }
            break;
        }
        case OP_PEXITEMDONE: {
            REQUIRE(m->role[t->actor] == R_PEX, "transition not enabled: actor");
            const int p = m->ordinal[t->actor];
            pex_t_* px = &s->pex[p];
            REQUIRE(px->pc == P_SENDITEMDONE, "transition not enabled: element item-done pc");
            unit_t_* un = &s->unit[pex_unit(m, p)];
            REQUIRE(un->pc == U_SERVE, "transition not enabled: unit serving");
            un->got_items += 1;
            memset(px, 0, sizeof *px);
            if (un->sent < m->wg)
                un->pc = U_REACTPEX;
            else if (m->kernel == 0 && un->got_items == m->wg)
                un->pc = U_SENDUNITDONE;
            break;
        }
        case OP_PEXENDDONE: {
            REQUIRE(m->role[t->actor] == R_PEX, "transition not enabled: actor");
            const int p = m->ordinal[t->actor];
            pex_t_* px = &s->pex[p];
            REQUIRE(px->pc == P_SENDENDDONE, "transition not enabled: element end-done pc");
            unit_t_* un = &s->unit[pex_unit(m, p)];
            REQUIRE(un->pc == U_SERVE, "transition not enabled: unit serving");
            un->got_ends += 1;
            if (pex_me(m, p) == 0) s->all_nwe -= 1;
            memset(px, 0, sizeof *px);
            if (un->got_ends == pl->nwe) un->pc = U_SENDUNITDONE;
            break;
        }
        default: m_fail(m, "transition not enabled: unknown op"); return;
    }
}

/* Machine::is_terminal, machine.cpp:651-662 */
static int is_terminal(const machine_t* m, const state_t* s) {
    if (!s->fin || s->clock != C_EXITED || s->host_pc != H_EXITED) return 0;
    for (int d = 0; d < m->plan.nwd; ++d)
        if (s->dev[d].pc != D_EXITED) return 0;
    for (int g = 0; g < m->n_units; ++g)
        if (s->unit[g].pc != U_EXITED || s->bar[g].pc != B_EXITED) return 0;
    for (int p = 0; p < m->n_pex; ++p)
        if (s->pex[p].pc != P_EXITED) return 0;
    return 1;
}

/* ------------------------------------------------------ serialization
 * Machine::serialize (machine.cpp:669-706) + hash64 (machine.cpp:24-34) */

typedef struct {
    unsigned char* b;
    size_t n, cap;
} bytes_t;

static void put(bytes_t* o, uint64_t v, int nbytes) {
    if (o->n + (size_t)nbytes > o->cap) {
        o->cap = (o->cap + (size_t)nbytes) * 2;
        o->b = (unsigned char*)realloc(o->b, o->cap);
    }
    for (int i = 0; i < nbytes; ++i) o->b[o->n++] = (unsigned char)((v >> (8 * i)) & 0xff);
}

static void serialize(const machine_t* m, const state_t* s, bytes_t* o) {
    o->n = 0;
    put(o, (uint64_t)s->time, 8);
    put(o, (uint32_t)s->nrp_work, 4);
    put(o, (uint32_t)s->all_nwe, 4);
    put(o, (uint64_t)s->fin, 1);
    put(o, (uint32_t)s->next_wg, 4);
    put(o, (uint64_t)s->host_pc, 1);
    put(o, (uint32_t)s->host_k, 4);
    put(o, (uint64_t)s->clock, 1);
    for (int d = 0; d < m->plan.nwd; ++d) {
        put(o, (uint64_t)s->dev[d].pc, 1);
        put(o, (uint32_t)s->dev[d].k, 4);
        put(o, (uint32_t)s->dev[d].batch_base, 4);
    }
    for (int g = 0; g < m->n_units; ++g) {
        const unit_t_* u = &s->unit[g];
        put(o, (uint64_t)u->pc, 1);
        put(o, (uint32_t)u->k, 4);
        put(o, (uint32_t)u->nwg, 4);
        put(o, (uint32_t)u->sent, 4);
        put(o, (uint32_t)u->got_items, 4);
        put(o, (uint32_t)u->got_ends, 4);
    }
    for (int g = 0; g < m->n_units; ++g) {
        put(o, (uint64_t)s->bar[g].pc, 1);
        put(o, (uint32_t)s->bar[g].count, 4);
    }
    for (int p = 0; p < m->n_pex; ++p) {
        const pex_t_* x = &s->pex[p];
        put(o, (uint64_t)x->pc, 1);
        put(o, (uint64_t)x->phase, 1);
        put(o, (uint32_t)x->cursor, 4);
        put(o, (uint32_t)x->busy_left, 4);
        put(o, (uint64_t)x->reported, 1);
        put(o, (uint32_t)x->nwg, 4);
        put(o, (uint32_t)x->iter, 4);
    }
    for (int i = 0; i < m->n_glob; ++i) put(o, (uint64_t)s->glob[i], 8);
    for (int i = 0; i < m->n_loc; ++i) put(o, (uint64_t)s->loc[i], 8);
}

static uint64_t hash64(const unsigned char* b, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ull;
    }
    h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ull;
    h = (h ^ (h >> 27)) * 0x94d049bb133111ebull;
    return h ^ (h >> 31);
}

/* ----------------------------------------------------------- RNGs */

/* std::mt19937_64 (the reference's SeededRandom policy, machine.cpp:791,807) */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64_t;

static void mt64_seed(mt64_t* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static uint64_t mt64_next(mt64_t* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

void mo_mt19937_64(uint64_t seed, int n, uint64_t* out) {
    mt64_t r;
    mt64_seed(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = mt64_next(&r);
}

/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) — the counter-based
 * generator of the swarm trajectories. */
void mo_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* Trajectory choice of the swarm: for trajectory `traj` under
 * `seed`, step i draws word i%4 of Philox(ctr={i/4, traj_lo, traj_hi, 0},
 * key={seed_lo, seed_hi}) and picks floor(word * n / 2^32). */
static int philox_pick(uint64_t seed, uint64_t traj, uint64_t step, int n) {
    const uint32_t ctr[4] = {(uint32_t)(step >> 2), (uint32_t)traj, (uint32_t)(traj >> 32),
                             (uint32_t)(step >> 34)};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    mo_philox4x32_10(ctr, key, out);
    return (int)(((uint64_t)out[step & 3] * (uint64_t)n) >> 32);
}

/* ------------------------------------------------------------- runs */

static int finish_bug(machine_t* m) {
    (void)m;
    return MO_MODEL_BUG;
}

/* Machine::run, machine.cpp:788-825 (+ our FIRST and PHILOX policies) */
int mo_simulate(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                int policy, uint64_t seed, uint64_t traj, int64_t* out, mo_transition* trace,
                int64_t cap, int64_t* trace_len) {
    const plat_t p = {plat[0], plat[1], plat[2], plat[3]};
    machine_t m;
    int rc = machine_init(&m, &p, size, kernel, input, wg, ts);
    if (rc) return rc;
    state_t s;
    state_alloc(&m, &s);
    initial_state(&m, &s);
    mt64_t rng;
    mt64_seed(&rng, seed);
    tvec en = {0};
    int64_t steps = 0;
    int rr_next = 0;
    const int64_t max_steps = 200000000LL; /* machine.hpp:215 kDefaultMaxRunSteps */
    rc = MO_OK;
    for (;;) {
        enabled(&m, &s, &en);
        if (en.n == 0) {
            if (is_terminal(&m, &s)) {
                out[0] = s.time;
                out[1] = steps;
                out[2] = kernel == 1 ? s.glob[0] : INT64_MIN;
                out[3] = m.n_proc;
                break;
            }
            m_fail(&m, "deadlock: non-terminal state with no enabled transition");
            rc = finish_bug(&m);
            break;
        }
        if (steps >= max_steps) {
            m_fail(&m, "run exceeded the step limit");
            rc = finish_bug(&m);
            break;
        }
        int pick = 0;
        if (policy == MO_POLICY_MT19937) {
            pick = (int)(mt64_next(&rng) % (uint64_t)en.n);
        } else if (policy == MO_POLICY_ROUND_ROBIN) {
            pick = en.n;
            for (int i = 0; i < en.n; ++i)
                if (en.v[i].actor >= rr_next) {
                    pick = i;
                    break;
                }
            if (pick == en.n) pick = 0;
            rr_next = (en.v[pick].actor + 1) % m.n_proc;
        } else if (policy == MO_POLICY_PHILOX) {
            pick = philox_pick(seed, traj, (uint64_t)steps, en.n);
        }
        if (trace && steps < cap) trace[steps] = en.v[pick];
        apply(&m, &s, &en.v[pick]);
        if (m.bug) {
            rc = MO_MODEL_BUG;
            break;
        }
        ++steps;
    }
    if (trace_len) *trace_len = steps;
    free(en.v);
    state_free(&s);
    machine_free(&m);
    return rc;
}

int mo_run_fingerprints(const int* plat, int size, int kernel, const int64_t* input, int wg,
                        int ts, const mo_transition* trace, int64_t len, uint64_t* out) {
    const plat_t p = {plat[0], plat[1], plat[2], plat[3]};
    machine_t m;
    int rc = machine_init(&m, &p, size, kernel, input, wg, ts);
    if (rc) return rc;
    state_t s;
    state_alloc(&m, &s);
    initial_state(&m, &s);
    bytes_t b = {0};
    serialize(&m, &s, &b);
    out[0] = hash64(b.b, b.n);
    for (int64_t i = 0; i < len && !rc; ++i) {
        apply(&m, &s, &trace[i]);
        if (m.bug) {
            rc = MO_MODEL_BUG;
            break;
        }
        serialize(&m, &s, &b);
        out[i + 1] = hash64(b.b, b.n);
    }
    free(b.b);
    state_free(&s);
    machine_free(&m);
    return rc;
}

/* replay, explore.cpp:283-300 */
int mo_replay(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
              const mo_transition* trace, int64_t len, int64_t final_time, int64_t* out) {
    const plat_t p = {plat[0], plat[1], plat[2], plat[3]};
    machine_t m;
    int rc = machine_init(&m, &p, size, kernel, input, wg, ts);
    if (rc) return rc;
    state_t s;
    state_alloc(&m, &s);
    initial_state(&m, &s);
    tvec en = {0};
    for (int64_t i = 0; i < len; ++i) {
        /* apply() enforces the guards of the op itself; a transition the
         * reference would reject is exactly one not in enabled(s). */
        enabled(&m, &s, &en);
        int found = 0;
        for (int j = 0; j < en.n && !found; ++j)
            found = en.v[j].actor == trace[i].actor && en.v[j].peer == trace[i].peer &&
                    en.v[j].op == trace[i].op;
        apply(&m, &s, &trace[i]);
        if (m.bug || !found) {
            set_err("replay diverged at step %lld", (long long)i);
            rc = MO_CORRUPT_TRACE;
            break;
        }
    }
    if (!rc && !is_terminal(&m, &s)) {
        set_err("replayed trace does not end terminal");
        rc = MO_CORRUPT_TRACE;
    }
    if (!rc && s.time != final_time) {
        set_err("replayed final time %lld != recorded %lld", (long long)s.time, (long long)final_time);
        rc = MO_CORRUPT_TRACE;
    }
    if (!rc) {
        out[0] = s.time;
        out[1] = kernel == 1 ? s.glob[0] : INT64_MIN;
    }
    free(en.v);
    state_free(&s);
    machine_free(&m);
    return rc;
}

/* Machine::label (machine.cpp:758-786) + process_name (machine.cpp:103-113) */
static int pname(const machine_t* m, int pid, char* buf, size_t n) {
    const int r = m->role[pid];
    if (r <= R_CLOCK) return snprintf(buf, n, "%s", ROLE_NAME[r]);
    return snprintf(buf, n, "%s%d", ROLE_NAME[r], m->ordinal[pid]);
}

static void label(const machine_t* m, const mo_transition* t, char* buf, size_t n) {
    char peer[64] = "";
    if (t->peer >= 0 && t->peer < m->n_proc) pname(m, t->peer, peer, sizeof peer);
    switch (t->op) {
        case OP_CLOCKTICK: snprintf(buf, n, "tick"); break;
        case OP_CLOCKHALT: snprintf(buf, n, "halt"); break;
        case OP_HOSTGO: snprintf(buf, n, "go -> %s", peer); break;
        case OP_HOSTREACTGO: snprintf(buf, n, "go(react) -> %s", peer); break;
        case OP_HOSTSTOP: snprintf(buf, n, "stop -> %s", peer); break;
        case OP_HOSTSETFIN: snprintf(buf, n, "fin"); break;
        case OP_DEVICEUNITGO: snprintf(buf, n, "go(wg%d) -> %s", t->arg, peer); break;
        case OP_DEVICEDONE: snprintf(buf, n, "done -> host"); break;
        case OP_DEVICEUNITSTOP: snprintf(buf, n, "stop -> %s", peer); break;
        case OP_UNITPEXGO: snprintf(buf, n, "go(round%d) -> %s", t->arg, peer); break;
        case OP_UNITDONE: snprintf(buf, n, "done(wg%d) -> %s", t->arg, peer); break;
        case OP_UNITPEXSTOP: snprintf(buf, n, "stop -> %s", peer); break;
        case OP_UNITBARRIERSTOP: snprintf(buf, n, "stop -> %s", peer); break;
        case OP_PEXREPORT: snprintf(buf, n, "report"); break;
        case OP_PEXEFFECT: snprintf(buf, n, "effect[%d]", t->arg); break;
        case OP_PEXARRIVE: snprintf(buf, n, "barrier-arrive -> %s", peer); break;
        case OP_PEXITEMDONE: snprintf(buf, n, "item-done -> %s", peer); break;
        case OP_PEXENDDONE: snprintf(buf, n, "group-done -> %s", peer); break;
        case OP_BARRIERRELEASE: snprintf(buf, n, "barrier-release"); break;
        default: snprintf(buf, n, "?"); break;
    }
}

/* trace_to_text, report.cpp:82-97 */
int64_t mo_trace_text(const int* plat, int size, int kernel, const int64_t* input, int wg,
                      int ts, const mo_transition* trace, int64_t len, char* buf, int64_t cap) {
    const plat_t p = {plat[0], plat[1], plat[2], plat[3]};
    machine_t m;
    if (machine_init(&m, &p, size, kernel, input, wg, ts)) return -1;
    state_t s;
    state_alloc(&m, &s);
    initial_state(&m, &s);
    bytes_t o = {0};
    char line[256], lab[128];
    for (int64_t i = 0; i < len; ++i) {
        apply(&m, &s, &trace[i]);
        if (m.bug) break;
        label(&m, &trace[i], lab, sizeof lab);
        const int k = snprintf(line, sizeof line, "%lld %d %s %s time=%lld\n", (long long)i,
                               trace[i].actor, ROLE_NAME[m.role[trace[i].actor]], lab,
                               (long long)s.time);
        for (int j = 0; j < k; ++j) put(&o, (unsigned char)line[j], 1);
    }
    int k = snprintf(line, sizeof line, "FINAL time=%lld wg=%d ts=%d", (long long)s.time, wg, ts);
    for (int j = 0; j < k; ++j) put(&o, (unsigned char)line[j], 1);
    if (kernel == 1) {
        k = snprintf(line, sizeof line, " result=%lld", (long long)s.glob[0]);
        for (int j = 0; j < k; ++j) put(&o, (unsigned char)line[j], 1);
    }
    put(&o, '\n', 1);
    const int64_t n = (int64_t)o.n;
    if (buf && cap > 0) {
        const int64_t c = n < cap - 1 ? n : cap - 1;
        memcpy(buf, o.b, (size_t)c);
        buf[c] = 0;
    }
    free(o.b);
    state_free(&s);
    machine_free(&m);
    return n;
}

/* ----------------------------------------------------------- explore
 * explore_machine (explore.cpp:86-165), exact mode: the visited set holds the
 * canonical serialization (explore.cpp:21-44). */

typedef struct {
    uint64_t* hash;
    unsigned char** key;
    uint32_t* len;
    size_t cap, n;
} vset_t;

static void vset_init(vset_t* v, size_t cap) {
    v->cap = cap;
    v->n = 0;
    v->hash = (uint64_t*)calloc(cap, sizeof(uint64_t));
    v->key = (unsigned char**)calloc(cap, sizeof(unsigned char*));
    v->len = (uint32_t*)calloc(cap, sizeof(uint32_t));
}

static void vset_free(vset_t* v) {
    for (size_t i = 0; i < v->cap; ++i) free(v->key[i]);
    free(v->hash);
    free(v->key);
    free(v->len);
}

static int vset_insert_raw(vset_t* v, const unsigned char* b, size_t n, uint64_t h);

static void vset_grow(vset_t* v) {
    vset_t nv;
    vset_init(&nv, v->cap * 2);
    for (size_t i = 0; i < v->cap; ++i)
        if (v->key[i]) {
            vset_insert_raw(&nv, v->key[i], v->len[i], v->hash[i]);
            free(v->key[i]);
            v->key[i] = NULL;
        }
    free(v->hash);
    free(v->key);
    free(v->len);
    *v = nv;
}

static int vset_insert_raw(vset_t* v, const unsigned char* b, size_t n, uint64_t h) {
    size_t i = (size_t)(h & (v->cap - 1));
    for (;;) {
        if (!v->key[i]) {
            v->key[i] = (unsigned char*)malloc(n);
            memcpy(v->key[i], b, n);
            v->len[i] = (uint32_t)n;
            v->hash[i] = h;
            v->n++;
            return 1;
        }
        if (v->hash[i] == h && v->len[i] == n && !memcmp(v->key[i], b, n)) return 0;
        i = (i + 1) & (v->cap - 1);
    }
}

static int vset_insert(vset_t* v, const unsigned char* b, size_t n) {
    if (2 * (v->n + 1) > v->cap) vset_grow(v);
    return vset_insert_raw(v, b, n, hash64(b, n));
}

typedef struct {
    state_t s;
    mo_transition* en;
    int n_en, next;
} node_t;

typedef struct {
    int64_t states, transitions, max_depth;
    int64_t min_t, max_t, n_term, n_distinct;
    int64_t distinct[64];
    int complete;
    /* first terminal with time <= T (T < 0: none wanted) */
    int64_t T;
    int found;
    int64_t found_time;
    mo_transition* trace;
    int64_t cap, trace_len;
} xres_t;

static int explore(machine_t* m, int64_t max_depth, int64_t max_states, xres_t* r) {
    vset_t vis;
    vset_init(&vis, 1 << 12);
    bytes_t b = {0};
    tvec en = {0};
    r->complete = 1;
    node_t* stack = NULL;
    int n_stack = 0, cap_stack = 0;
    mo_transition* path = NULL;
    int64_t n_path = 0, cap_path = 0;
    int rc = MO_OK;

    state_t init;
    state_alloc(m, &init);
    initial_state(m, &init);
    serialize(m, &init, &b);
    vset_insert(&vis, b.b, b.n);
    r->states += 1;
    enabled(m, &init, &en);
    if (en.n == 0) {
        set_err("initial state has no enabled transitions");
        state_free(&init);
        free(b.b);
        free(en.v);
        vset_free(&vis);
        return MO_MODEL_BUG;
    }
    cap_stack = 64;
    stack = (node_t*)malloc(sizeof(node_t) * (size_t)cap_stack);
    stack[0].s = init;
    stack[0].en = (mo_transition*)malloc(sizeof(mo_transition) * (size_t)en.n);
    memcpy(stack[0].en, en.v, sizeof(mo_transition) * (size_t)en.n);
    stack[0].n_en = en.n;
    stack[0].next = 0;
    n_stack = 1;

    while (n_stack > 0) {
        node_t* node = &stack[n_stack - 1];
        if (node->next >= node->n_en) {
            state_free(&node->s);
            free(node->en);
            --n_stack;
            if (n_path > 0) --n_path;
            continue;
        }
        const mo_transition t = node->en[node->next++];
        if (n_path + 1 > max_depth) {
            r->complete = 0;
            continue;
        }
        state_t succ;
        state_alloc(m, &succ);
        state_copy(m, &succ, &node->s);
        apply(m, &succ, &t);
        if (m->bug) {
            state_free(&succ);
            rc = MO_MODEL_BUG;
            break;
        }
        r->transitions += 1;
        serialize(m, &succ, &b);
        int ins;
        if ((int64_t)vis.n >= max_states)
            ins = -1;
        else
            ins = vset_insert(&vis, b.b, b.n);
        if (ins <= 0) {
            if (ins < 0) r->complete = 0;
            state_free(&succ);
            continue;
        }
        r->states += 1;
        if (n_path + 1 > r->max_depth) r->max_depth = n_path + 1;
        enabled(m, &succ, &en);
        if (n_path + 1 > cap_path) {
            cap_path = cap_path ? 2 * cap_path : 1024;
            path = (mo_transition*)realloc(path, sizeof(mo_transition) * (size_t)cap_path);
        }
        if (en.n == 0) {
            if (!is_terminal(m, &succ)) {
                set_err("deadlock reached");
                state_free(&succ);
                rc = MO_MODEL_BUG;
                break;
            }
            r->n_term += 1;
            if (r->min_t < 0 || succ.time < r->min_t) r->min_t = succ.time;
            if (succ.time > r->max_t) r->max_t = succ.time;
            int seen = 0;
            for (int64_t i = 0; i < r->n_distinct && i < 64; ++i) seen |= r->distinct[i] == succ.time;
            if (!seen) {
                if (r->n_distinct < 64) r->distinct[r->n_distinct] = succ.time;
                r->n_distinct++;
            }
            if (r->T >= 0 && succ.time <= r->T) {
                path[n_path] = t;
                r->found = 1;
                r->found_time = succ.time;
                r->trace_len = n_path + 1;
                if (r->trace)
                    memcpy(r->trace, path,
                           sizeof(mo_transition) * (size_t)(r->trace_len < r->cap ? r->trace_len : r->cap));
                state_free(&succ);
                break;
            }
            state_free(&succ);
            continue;
        }
        path[n_path++] = t;
        if (n_stack == cap_stack) {
            cap_stack *= 2;
            stack = (node_t*)realloc(stack, sizeof(node_t) * (size_t)cap_stack);
        }
        stack[n_stack].s = succ;
        stack[n_stack].en = (mo_transition*)malloc(sizeof(mo_transition) * (size_t)en.n);
        memcpy(stack[n_stack].en, en.v, sizeof(mo_transition) * (size_t)en.n);
        stack[n_stack].n_en = en.n;
        stack[n_stack].next = 0;
        ++n_stack;
    }
    for (int i = 0; i < n_stack; ++i) {
        state_free(&stack[i].s);
        free(stack[i].en);
    }
    free(stack);
    free(path);
    free(b.b);
    free(en.v);
    vset_free(&vis);
    return rc;
}

int mo_explore(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
               int64_t max_depth, int64_t max_states, int64_t* out) {
    const plat_t p = {plat[0], plat[1], plat[2], plat[3]};
    machine_t m;
    int rc = machine_init(&m, &p, size, kernel, input, wg, ts);
    if (rc) return rc;
    xres_t r;
    memset(&r, 0, sizeof r);
    r.min_t = -1;
    r.max_t = -1;
    r.T = -1;
    rc = explore(&m, max_depth > 0 ? max_depth : 4000000, max_states > 0 ? max_states : 5000000, &r);
    out[0] = r.complete;
    out[1] = r.states;
    out[2] = r.transitions;
    out[3] = r.max_depth;
    out[4] = r.min_t;
    out[5] = r.max_t;
    out[6] = r.n_term;
    out[7] = r.n_distinct;
    machine_free(&m);
    return rc;
}

/* check_overtime, explore.cpp:167-205 (exact mode) */
int mo_check_overtime(const int* plat, int size, int kernel, const int64_t* input, int64_t T,
                      int64_t max_depth, int64_t max_states, int64_t* out, mo_transition* trace,
                      int64_t cap, int64_t* trace_len) {
    if (T < 0) {
        set_err("over-time bound must be >= 0");
        return MO_CONFIG_ERROR;
    }
    const plat_t p = {plat[0], plat[1], plat[2], plat[3]};
    int rc = validate_platform(&p);
    if (rc) return rc;
    if (size < 4 || !is_pow2(size)) {
        set_err("size must be a power of two >= 4");
        return MO_CONFIG_ERROR;
    }
    const int n = log2i(size);
    int64_t states = 0, trans = 0, maxd = 0, explored = 0, skipped = 0;
    int limit_hit = 0, violated = 0;
    for (int i = 0; i < 11; ++i) out[i] = 0;
    out[7] = -1;
    if (trace_len) *trace_len = 0;
    /* feasible configs sorted (wg desc, ts desc), explore.cpp:52-72; skipped
     * configurations are counted up front (explore.cpp:52-62) */
    for (int i = 1; i <= n - 1; ++i)
        for (int j = 1; j <= n - 1; ++j)
            if (kernel == 1 && (1LL << (i + j)) > size) ++skipped;
    for (int i = n - 1; i >= 1 && !violated; --i)
        for (int j = n - 1; j >= 1 && !violated; --j) {
            const int wg = 1 << i, ts = 1 << j;
            if (kernel == 1 && (long long)wg * ts > size) continue;
            machine_t m;
            if ((rc = machine_init(&m, &p, size, kernel, input, wg, ts))) return rc;
            ++explored;
            xres_t r;
            memset(&r, 0, sizeof r);
            r.min_t = -1;
            r.max_t = -1;
            r.T = T;
            r.trace = trace;
            r.cap = cap;
            rc = explore(&m, max_depth > 0 ? max_depth : 4000000,
                         max_states > 0 ? max_states : 5000000, &r);
            machine_free(&m);
            if (rc) return rc;
            states += r.states;
            trans += r.transitions;
            if (r.max_depth > maxd) maxd = r.max_depth;
            if (!r.complete) limit_hit = 1;
            if (r.found) {
                violated = 1;
                out[7] = r.found_time;
                out[8] = wg;
                out[9] = ts;
                out[10] = r.trace_len;
                if (trace_len) *trace_len = r.trace_len;
            }
        }
    out[0] = violated;
    out[1] = !violated && !limit_hit;
    out[2] = states;
    out[3] = maxd;
    out[4] = trans;
    out[5] = explored;
    out[6] = skipped;
    return MO_OK;
}

/* -------------------------------------------------- generalised space
 * Space descriptor (int64 x 13), DESIGN.md §4 / include/mctune_b200.h:
 *  [0] kernel [1] size [2] gmt [3] nd_lo [4] nd_hi [5] nu_lo [6] nu_hi
 *  [7] lognp_lo [8] lognp_hi [9] logwg_lo [10] logwg_hi [11] logts_lo [12] logts_hi
 * index = ((((wg_d * Nts + ts_d) * Nnp + np_d) * Nnu + nu_d) * Nnd + nd_d)
 * with wg_d = logwg_hi - logwg, ts_d = logts_hi - logts (descending: the
 * reference's tie preference, explore.cpp:64-72), np/nu/nd ascending. */

int mo_space_decode(const int64_t* sd, uint64_t index, int* cfg) {
    const uint64_t Nnd = (uint64_t)(sd[4] - sd[3] + 1), Nnu = (uint64_t)(sd[6] - sd[5] + 1),
                   Nnp = (uint64_t)(sd[8] - sd[7] + 1), Nts = (uint64_t)(sd[12] - sd[11] + 1);
    const uint64_t nd_d = index % Nnd;
    index /= Nnd;
    const uint64_t nu_d = index % Nnu;
    index /= Nnu;
    const uint64_t np_d = index % Nnp;
    index /= Nnp;
    const uint64_t ts_d = index % Nts;
    const uint64_t wg_d = index / Nts;
    cfg[0] = (int)(sd[3] + (int64_t)nd_d);
    cfg[1] = (int)(sd[5] + (int64_t)nu_d);
    cfg[2] = 1 << (int)(sd[7] + (int64_t)np_d);
    cfg[3] = (int)sd[2];
    cfg[4] = (int)sd[1];
    cfg[5] = (int)sd[0];
    cfg[6] = 1 << (int)(sd[10] - (int64_t)wg_d);
    cfg[7] = 1 << (int)(sd[12] - (int64_t)ts_d);
    return MO_OK;
}

#define MO_KEY_TIME_BITS 30
#define MO_KEY_INDEX_BITS 33

/* Exact argmin of [first, first+count): the least (time, index) over the feasible
 * configurations — the reference's tie rule (search.cpp:67-78: least time, then
 * the preferred configuration, which the index order puts first).  best_time = -1
 * and best_index = UINT64_MAX when the range holds no feasible configuration.
 * best_key is the GPU's packed key of the range, (min(time, 2^30-1) << 33) | index
 * minimised over every configuration (infeasible ones carry the saturated time):
 * exact only while its time field is below 2^30-1, which is why best_time and
 * best_index are computed without it. */
int mo_space_argmin(const int64_t* sd, uint64_t first, uint64_t count, uint64_t* best_key,
                    int64_t* best_time, uint64_t* best_index) {
    uint64_t best = UINT64_MAX, bi = UINT64_MAX;
    int64_t bt = -1;
    const uint64_t sat = (1ull << MO_KEY_TIME_BITS) - 1;
    for (uint64_t i = first; i < first + count; ++i) {
        int c[8];
        mo_space_decode(sd, i, c);
        const plat_t p = {c[0], c[1], c[2], c[3]};
        uint64_t tf = sat;
        if (!(c[5] == 1 && (long long)c[6] * c[7] > c[4])) {
            int64_t t, st;
            cost_model(&p, c[4], c[5], c[6], c[7], &t, &st);
            tf = (uint64_t)t < sat ? (uint64_t)t : sat;
            if (bt < 0 || t < bt) { /* ascending index: the first of equal times stays */
                bt = t;
                bi = i;
            }
        }
        const uint64_t key = (tf << MO_KEY_INDEX_BITS) | i;
        if (key < best) best = key;
    }
    *best_key = best;
    *best_time = bt;
    *best_index = bi;
    return MO_OK;
}

/* Bulk CPU replay of GPU trajectories (checker for mctb_trajectories):
 * trajectory t = traj0 + i runs configs[t % n_configs] under `policy`;
 * out = int64[6 * n]: {time, steps, result, status, FNV-1a 64 over the trace's
 * 32-bit words, config}. */
static uint64_t fnv_words(uint64_t h, const mo_transition* t) {
    /* FNV-1a over the four 32-bit words (one xor-multiply per word) */
    const int32_t w[4] = {t->actor, t->peer, t->op, t->arg};
    for (int k = 0; k < 4; ++k) {
        h ^= (uint32_t)w[k];
        h *= 0x100000001b3ull;
    }
    return h;
}

int mo_trajectories(const int* plat, int size, int kernel, const int64_t* input,
                    const int32_t* configs, int n_configs, int policy, uint64_t seed,
                    uint64_t traj0, uint64_t n, int64_t* out) {
    int64_t cap = 1 << 20;
    mo_transition* tr = (mo_transition*)malloc(sizeof(mo_transition) * (size_t)cap);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t t = traj0 + i;
        const int c = (int)(t % (uint64_t)n_configs);
        int64_t o[4], len = 0;
        int rc = mo_simulate(plat, size, kernel, input, configs[2 * c], configs[2 * c + 1], policy,
                             seed, t, o, tr, cap, &len);
        if (rc == MO_OK && len > cap) {
            cap = len;
            tr = (mo_transition*)realloc(tr, sizeof(mo_transition) * (size_t)cap);
            rc = mo_simulate(plat, size, kernel, input, configs[2 * c], configs[2 * c + 1], policy,
                             seed, t, o, tr, cap, &len);
        }
        if (rc) {
            free(tr);
            return rc;
        }
        uint64_t h = 0xcbf29ce484222325ull;
        for (int64_t k = 0; k < len; ++k) h = fnv_words(h, &tr[k]);
        int64_t* r = out + 6 * i;
        r[0] = o[0];
        r[1] = o[1];
        r[2] = o[2];
        r[3] = 0;
        r[4] = (int64_t)h;
        r[5] = c;
    }
    free(tr);
    return MO_OK;
}

/* ------------------------------------------------- successor enumeration
 * For the multi-rank exploration test (tests/test_distributed.py): states are
 * exchanged in the reference's canonical serialization (machine.cpp:669-706). */
static uint64_t get_le(const unsigned char** p, int nbytes) {
    uint64_t v = 0;
    for (int i = 0; i < nbytes; ++i) v |= (uint64_t)(*p)[i] << (8 * i);
    *p += nbytes;
    return v;
}

static void deserialize(const machine_t* m, const unsigned char* b, state_t* s) {
    const unsigned char* p = b;
    s->time = (int64_t)get_le(&p, 8);
    s->nrp_work = (int32_t)get_le(&p, 4);
    s->all_nwe = (int32_t)get_le(&p, 4);
    s->fin = (int32_t)get_le(&p, 1);
    s->next_wg = (int32_t)get_le(&p, 4);
    s->host_pc = (int32_t)get_le(&p, 1);
    s->host_k = (int32_t)get_le(&p, 4);
    s->clock = (int32_t)get_le(&p, 1);
    for (int d = 0; d < m->plan.nwd; ++d) {
        s->dev[d].pc = (int32_t)get_le(&p, 1);
        s->dev[d].k = (int32_t)get_le(&p, 4);
        s->dev[d].batch_base = (int32_t)get_le(&p, 4);
    }
    for (int g = 0; g < m->n_units; ++g) {
        unit_t_* u = &s->unit[g];
        u->pc = (int32_t)get_le(&p, 1);
        u->k = (int32_t)get_le(&p, 4);
        u->nwg = (int32_t)get_le(&p, 4);
        u->sent = (int32_t)get_le(&p, 4);
        u->got_items = (int32_t)get_le(&p, 4);
        u->got_ends = (int32_t)get_le(&p, 4);
    }
    for (int g = 0; g < m->n_units; ++g) {
        s->bar[g].pc = (int32_t)get_le(&p, 1);
        s->bar[g].count = (int32_t)get_le(&p, 4);
    }
    for (int q = 0; q < m->n_pex; ++q) {
        pex_t_* x = &s->pex[q];
        x->pc = (int32_t)get_le(&p, 1);
        x->phase = (int32_t)get_le(&p, 1);
        x->cursor = (int32_t)get_le(&p, 4);
        x->busy_left = (int32_t)get_le(&p, 4);
        x->reported = (int32_t)get_le(&p, 1);
        x->nwg = (int32_t)get_le(&p, 4);
        x->iter = (int32_t)get_le(&p, 4);
    }
    for (int i = 0; i < m->n_glob; ++i) s->glob[i] = (int64_t)get_le(&p, 8);
    for (int i = 0; i < m->n_loc; ++i) s->loc[i] = (int64_t)get_le(&p, 8);
}

/* Serialization of the initial state (ser == NULL) or of every successor of the
 * serialized state `ser`; out receives n records of `*rec_len` bytes and
 * fps[i] = hash64 (the reference's fingerprint).  Returns the record count. */
int64_t mo_successors(const int* plat, int size, int kernel, const int64_t* input, int wg, int ts,
                      const unsigned char* ser, unsigned char* out, int64_t cap, uint64_t* fps,
                      int64_t* rec_len) {
    const plat_t p = {plat[0], plat[1], plat[2], plat[3]};
    machine_t m;
    if (machine_init(&m, &p, size, kernel, input, wg, ts)) return -1;
    state_t s, t;
    state_alloc(&m, &s);
    state_alloc(&m, &t);
    initial_state(&m, &s);
    bytes_t b = {0};
    int64_t n = 0;
    if (!ser) {
        serialize(&m, &s, &b);
        *rec_len = (int64_t)b.n;
        if (cap >= 1) {
            memcpy(out, b.b, b.n);
            fps[0] = hash64(b.b, b.n);
        }
        n = 1;
    } else {
        deserialize(&m, ser, &s);
        tvec en = {0};
        enabled(&m, &s, &en);
        for (int i = 0; i < en.n; ++i) {
            state_copy(&m, &t, &s);
            apply(&m, &t, &en.v[i]);
            serialize(&m, &t, &b);
            *rec_len = (int64_t)b.n;
            if (n < cap) {
                memcpy(out + n * b.n, b.b, b.n);
                fps[n] = hash64(b.b, b.n);
            }
            ++n;
        }
        free(en.v);
    }
    free(b.b);
    state_free(&s);
    state_free(&t);
    const int bug = m.bug;
    machine_free(&m);
    return bug ? -1 : n;
}
