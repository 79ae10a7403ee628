/* TEST INFRASTRUCTURE ONLY — an independent CPU count of a configuration's
 * reachable states and transitions, to pin the GPU exploration on spaces too
 * large for the reference's DFS (whose visited set of serialized strings needs
 * more memory than this host has for 1.4e8 states).
 *
 * Level-synchronous BFS over the oracle's successor function (mo_successors:
 * machine.cpp:174-649 restated in mctune_oracle.c, pinned against the reference
 * in tests/test_oracle.py), on all host threads.  The visited set keeps a
 * 128-bit fingerprint of each canonical serialization (two independent 64-bit
 * hashes): a false "already visited" needs a 128-bit collision, probability
 * ~n^2 / 2^129 < 1e-22 at n = 1.4e8.  Prints {states, transitions, levels,
 * terminals}.  Build/run: see oracle/Makefile (count_states).
 */
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mctune_oracle.h"

static int g_plat[4], g_size, g_kernel, g_wg, g_ts;
static int64_t g_len;  /* serialized record length */
static _Atomic uint64_t* g_h1;
static _Atomic uint64_t* g_h2;
static uint64_t g_mask;

static uint64_t mix(uint64_t h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdULL;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ULL;
    h ^= h >> 33;
    return h;
}

static void fp128(const unsigned char* b, int64_t n, uint64_t* a, uint64_t* c) {
    uint64_t x = 0x9e3779b97f4a7c15ULL, y = 0xcbf29ce484222325ULL;
    for (int64_t i = 0; i < n; ++i) {
        x = (x ^ b[i]) * 0x100000001b3ULL;
        y = mix(y + b[i] + 0x632be59bd9b4e019ULL * (uint64_t)(i + 1));
    }
    *a = mix(x) | 1ULL;
    *c = mix(y ^ (x << 1)) | 1ULL;
}

/* 1 = inserted, 0 = present */
static int insert(uint64_t a, uint64_t c) {
    uint64_t i = a & g_mask;
    for (;;) {
        uint64_t cur = atomic_load_explicit(&g_h1[i], memory_order_acquire);
        if (cur == 0) {
            uint64_t z = 0;
            if (atomic_compare_exchange_strong(&g_h1[i], &z, a)) {
                atomic_store_explicit(&g_h2[i], c, memory_order_release);
                return 1;
            }
            cur = z;
        }
        if (cur == a) {
            uint64_t d;
            while ((d = atomic_load_explicit(&g_h2[i], memory_order_acquire)) == 0) {
            }
            if (d == c) return 0;
        }
        i = (i + 1) & g_mask;
    }
}

typedef struct {
    const unsigned char* in;
    int64_t lo, hi;
    unsigned char* out;
    int64_t n_out, cap_out;
    int64_t transitions, terminals;
} work_t;

static void* expand(void* arg) {
    work_t* w = (work_t*)arg;
    unsigned char* buf = malloc(256 * g_len);
    uint64_t fps[256];
    for (int64_t k = w->lo; k < w->hi; ++k) {
        int64_t rl = 0;
        const int64_t n = mo_successors(g_plat, g_size, g_kernel, NULL, g_wg, g_ts,
                                        w->in + k * g_len, buf, 256, fps, &rl);
        if (n < 0 || n > 256) {
            fprintf(stderr, "successor error\n");
            exit(2);
        }
        if (n == 0) w->terminals += 1;
        w->transitions += n;
        for (int64_t e = 0; e < n; ++e) {
            uint64_t a, c;
            fp128(buf + e * g_len, g_len, &a, &c);
            if (insert(a, c)) {
                if (w->n_out == w->cap_out) {
                    w->cap_out = w->cap_out ? 2 * w->cap_out : 4096;
                    w->out = realloc(w->out, w->cap_out * g_len);
                }
                memcpy(w->out + w->n_out * g_len, buf + e * g_len, g_len);
                w->n_out += 1;
            }
        }
    }
    free(buf);
    return NULL;
}

int main(int argc, char** argv) {
    if (argc < 10) {
        fprintf(stderr, "usage: count_states nd nu np gmt size kernel wg ts log2slots [threads]\n");
        return 1;
    }
    for (int i = 0; i < 4; ++i) g_plat[i] = atoi(argv[1 + i]);
    g_size = atoi(argv[5]);
    g_kernel = atoi(argv[6]);
    g_wg = atoi(argv[7]);
    g_ts = atoi(argv[8]);
    const int lg = atoi(argv[9]);
    const int T = argc > 10 ? atoi(argv[10]) : 8;
    g_mask = (1ULL << lg) - 1;
    g_h1 = calloc(1ULL << lg, 8);
    g_h2 = calloc(1ULL << lg, 8);
    unsigned char init[65536];
    uint64_t fp;
    if (mo_successors(g_plat, g_size, g_kernel, NULL, g_wg, g_ts, NULL, init, 1, &fp, &g_len) != 1) {
        fprintf(stderr, "initial state error\n");
        return 2;
    }
    uint64_t a, c;
    fp128(init, g_len, &a, &c);
    insert(a, c);
    unsigned char* cur = malloc(g_len);
    memcpy(cur, init, g_len);
    int64_t n_cur = 1, states = 1, transitions = 0, terminals = 0, levels = 0;
    while (n_cur > 0) {
        work_t* w = calloc(T, sizeof(work_t));
        pthread_t th[256];
        for (int t = 0; t < T; ++t) {
            w[t].in = cur;
            w[t].lo = n_cur * t / T;
            w[t].hi = n_cur * (t + 1) / T;
            pthread_create(&th[t], NULL, expand, &w[t]);
        }
        int64_t n_next = 0;
        for (int t = 0; t < T; ++t) {
            pthread_join(th[t], NULL);
            n_next += w[t].n_out;
            transitions += w[t].transitions;
            terminals += w[t].terminals;
        }
        free(cur);
        cur = malloc((n_next ? n_next : 1) * g_len);
        int64_t pos = 0;
        for (int t = 0; t < T; ++t) {
            memcpy(cur + pos * g_len, w[t].out, w[t].n_out * g_len);
            pos += w[t].n_out;
            free(w[t].out);
        }
        free(w);
        n_cur = n_next;
        states += n_next;
        levels += 1;
        if (states > (int64_t)(g_mask / 10 * 7)) {
            fprintf(stderr, "fingerprint table too small\n");
            return 3;
        }
    }
    printf("{\"states\": %lld, \"transitions\": %lld, \"levels\": %lld, \"terminals\": %lld}\n",
           (long long)states, (long long)transitions, (long long)levels, (long long)terminals);
    return 0;
}
