/*
 * Seeded synthetic inputs for the five BASELINE.json configurations
 * (SURVEY.md Appendix A). The reference's own generator
 * (proj/src/generator.hpp:91-132) draws with replacement and never yields the
 * distinct keys the bitset sort needs, so only its PRNG is reused:
 * splitmix64 (generator.hpp:21-30), seed 42 for every config.
 *
 *   C1/C2  bws_gen_shuffle_prefix   forward Fisher-Yates prefix of [0, M):
 *                                   j = i + next() % (M - i); swap(p[i], p[j])
 *   C3     bws_gen_permutation      keyed Feistel bijection of [0, n) (the
 *                                   faster alternative Appendix A.3 allows for
 *                                   a full 2^30 permutation; parallel)
 *   C4     bws_gen_dedup_draws      (uint32)next() draws, first occurrences,
 *                                   draw order kept
 *   C5     bws_gen_clustered        4096 splitmix64 centres, Zipf(s) weights by
 *                                   generation rank, water-filled to the
 *                                   +-half_window capacity with largest-
 *                                   remainder rounding; per cluster a partial
 *                                   Fisher-Yates over the window's free keys
 *                                   (spilling any shortfall to the next rank);
 *                                   finally a Feistel shuffle of positions
 *
 * These are data generators (bench + tests), not the sort; they run on the
 * host, with pthreads where the recipe is parallel.
 */
#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GEN_API __attribute__((visibility("default")))

static inline uint64_t sm64_next(uint64_t* s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}


/* ---- minimal pthread parallel-for over [0, n) ---- */
typedef void (*range_fn)(void* ctx, uint64_t begin, uint64_t end);
typedef struct {
    range_fn fn;
    void* ctx;
    uint64_t begin, end;
} range_job;

static void* range_thread(void* arg) {
    range_job* j = (range_job*)arg;
    j->fn(j->ctx, j->begin, j->end);
    return NULL;
}

static void parallel_for(uint64_t n, range_fn fn, void* ctx) {
    long nt = sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if (nt > 64) nt = 64;
    if (n < (1ull << 16)) nt = 1;
    pthread_t th[64];
    range_job jobs[64];
    long started = 0;
    for (long t = 0; t < nt; ++t) {
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].begin = n * (uint64_t)t / (uint64_t)nt;
        jobs[t].end = n * (uint64_t)(t + 1) / (uint64_t)nt;
        if (t == nt - 1 || pthread_create(&th[t], NULL, range_thread, &jobs[t]) != 0) {
            range_thread(&jobs[t]);
        } else {
            ++started;
        }
    }
    for (long t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

GEN_API uint64_t bws_gen_fnv1a64(const void* data, size_t bytes) {
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < bytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

static void iota_range(void* ctx, uint64_t b, uint64_t e) {
    uint32_t* p = (uint32_t*)ctx;
    for (uint64_t i = b; i < e; ++i) p[i] = (uint32_t)i;
}

/* C1, C2: first n entries of a forward Fisher-Yates shuffle of [0, M). */
GEN_API int bws_gen_shuffle_prefix(uint32_t* out, uint64_t n, uint64_t M, uint64_t seed) {
    if (n > M || M > (1ull << 32)) return -2;
    uint32_t* p = (uint32_t*)malloc(M * sizeof(uint32_t));
    if (!p) return -1;
    parallel_for(M, iota_range, p);
    uint64_t s = seed;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t j = i + sm64_next(&s) % (M - i);
        const uint32_t t = p[i];
        p[i] = p[j];
        p[j] = t;
    }
    memcpy(out, p, n * sizeof(uint32_t));
    free(p);
    return 0;
}

/* Keyed Feistel network on 2h bits (h <= 32), 6 rounds, round keys from
 * splitmix64{seed}; cycle-walked into [0, n). */
typedef struct {
    unsigned half;
    uint64_t mask;
    uint64_t keys[6];
    uint64_t n;
} feistel_t;

static void feistel_init(feistel_t* f, uint64_t n, uint64_t seed) {
    unsigned bits = 2;
    while (bits < 64 && (1ull << bits) < n) ++bits;
    if (bits & 1) ++bits;
    f->half = bits / 2;
    f->mask = (1ull << f->half) - 1;
    uint64_t s = seed;
    for (int r = 0; r < 6; ++r) f->keys[r] = sm64_next(&s);
    f->n = n;
}

static inline uint64_t feistel_round(uint64_t x, uint64_t k) {
    uint64_t z = (x ^ k) + 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static inline uint64_t feistel_apply(const feistel_t* f, uint64_t x) {
    do {
        uint64_t l = x >> f->half, r = x & f->mask;
        for (int i = 0; i < 6; ++i) {
            const uint64_t t = l ^ (feistel_round(r, f->keys[i]) & f->mask);
            l = r;
            r = t;
        }
        x = (l << f->half) | r;
    } while (x >= f->n);
    return x;
}

typedef struct {
    const feistel_t* f;
    uint32_t* out;
    const uint32_t* src; /* NULL: out[i] = P(i); else out[P(i)] = src[i] */
} perm_ctx;

static void perm_range(void* ctx, uint64_t b, uint64_t e) {
    perm_ctx* c = (perm_ctx*)ctx;
    if (c->src) {
        for (uint64_t i = b; i < e; ++i) c->out[feistel_apply(c->f, i)] = c->src[i];
    } else {
        for (uint64_t i = b; i < e; ++i) c->out[i] = (uint32_t)feistel_apply(c->f, i);
    }
}

/* C3: out[i] = P(i), P a seeded pseudo-random permutation of [0, n). */
GEN_API int bws_gen_permutation(uint32_t* out, uint64_t n, uint64_t seed) {
    if (n > (1ull << 32)) return -2;
    feistel_t f;
    feistel_init(&f, n, seed);
    perm_ctx c = {&f, out, NULL};
    parallel_for(n, perm_range, &c);
    return 0;
}

/* C4: n distinct (uint32)next() draws in draw order. */
GEN_API int bws_gen_dedup_draws(uint32_t* out, uint64_t n, uint64_t seed) {
    if (n > (1ull << 32)) return -2;
    uint64_t* seen = (uint64_t*)calloc((1ull << 32) / 64, sizeof(uint64_t));
    if (!seen) return -1;
    uint64_t s = seed, k = 0;
    while (k < n) {
        const uint32_t x = (uint32_t)sm64_next(&s);
        const uint64_t bit = 1ull << (x & 63);
        if (seen[x >> 6] & bit) continue;
        seen[x >> 6] |= bit;
        out[k++] = x;
    }
    free(seen);
    return 0;
}

/* Cluster sizes for C5: s_k = min(cap_k, lambda * k^-zipf_s), sum exactly n
 * (water-filling, then largest-remainder rounding of the uncapped clusters;
 * ties go to the lower rank). Returns 0, or -3 if the windows cannot hold n. */
GEN_API int bws_gen_cluster_sizes(uint64_t* sizes, const uint64_t* caps, uint32_t clusters,
                                  uint64_t n, double zipf_s) {
    double* w = (double*)malloc(clusters * sizeof(double));
    unsigned char* capped = (unsigned char*)calloc(clusters, 1);
    double* frac = (double*)malloc(clusters * sizeof(double));
    if (!w || !capped || !frac) {
        free(w);
        free(capped);
        free(frac);
        return -1;
    }
    uint64_t cap_total = 0;
    for (uint32_t k = 0; k < clusters; ++k) {
        w[k] = pow((double)(k + 1), -zipf_s);
        cap_total += caps[k];
    }
    if (cap_total < n) {
        free(w);
        free(capped);
        free(frac);
        return -3;
    }
    double lambda = 0;
    for (;;) {
        double wsum = 0;
        uint64_t fixed = 0;
        for (uint32_t k = 0; k < clusters; ++k) {
            if (capped[k])
                fixed += caps[k];
            else
                wsum += w[k];
        }
        lambda = wsum > 0 ? (double)(n - fixed) / wsum : 0;
        int changed = 0;
        for (uint32_t k = 0; k < clusters; ++k) {
            if (!capped[k] && lambda * w[k] >= (double)caps[k]) {
                capped[k] = 1;
                changed = 1;
            }
        }
        if (!changed) break;
    }
    uint64_t assigned = 0;
    for (uint32_t k = 0; k < clusters; ++k) {
        if (capped[k]) {
            sizes[k] = caps[k];
            frac[k] = -1;
        } else {
            const double t = lambda * w[k];
            sizes[k] = (uint64_t)floor(t);
            frac[k] = t - floor(t);
        }
        assigned += sizes[k];
    }
    while (assigned < n) {
        uint32_t best = 0;
        double bf = -2;
        for (uint32_t k = 0; k < clusters; ++k)
            if (frac[k] > bf && sizes[k] < caps[k]) {
                bf = frac[k];
                best = k;
            }
        sizes[best] += 1;
        frac[best] = -1;
        ++assigned;
    }
    free(w);
    free(capped);
    free(frac);
    return 0;
}

/* C5: clustered distinct keys, shuffled. `centres_out` (optional) receives the
 * `clusters` centres in generation order. */
GEN_API int bws_gen_clustered(uint32_t* out, uint64_t n, uint32_t clusters, double zipf_s,
                              uint64_t half_window, uint64_t seed, uint32_t* centres_out) {
    if (n > (1ull << 32) || clusters == 0) return -2;
    uint64_t s = seed;
    uint64_t* lo = (uint64_t*)malloc(clusters * sizeof(uint64_t));
    uint64_t* caps = (uint64_t*)malloc(clusters * sizeof(uint64_t));
    uint64_t* sizes = (uint64_t*)malloc(clusters * sizeof(uint64_t));
    uint64_t* taken = (uint64_t*)calloc((1ull << 32) / 64, sizeof(uint64_t));
    uint32_t* freelist = (uint32_t*)malloc((2 * half_window + 1) * sizeof(uint32_t));
    uint32_t* tmp = (uint32_t*)malloc(n * sizeof(uint32_t));
    int rc = 0;
    if (!lo || !caps || !sizes || !taken || !freelist || !tmp) {
        rc = -1;
        goto done;
    }
    for (uint32_t k = 0; k < clusters; ++k) {
        const uint64_t c = (uint32_t)sm64_next(&s);
        if (centres_out) centres_out[k] = (uint32_t)c;
        const uint64_t a = c >= half_window ? c - half_window : 0;
        const uint64_t b = c + half_window <= 0xffffffffull ? c + half_window : 0xffffffffull;
        lo[k] = a;
        caps[k] = b - a + 1;
    }
    rc = bws_gen_cluster_sizes(sizes, caps, clusters, n, zipf_s);
    if (rc != 0) goto done;
    {
        uint64_t filled = 0, carry = 0;
        /* rank order; a window short of free keys spills to the next rank,
         * wrapping once around the cluster list */
        for (uint64_t step = 0; step < 2ull * clusters && filled < n; ++step) {
            const uint32_t k = (uint32_t)(step % clusters);
            uint64_t want = (step < clusters ? sizes[k] : 0) + carry;
            if (want == 0) continue;
            uint64_t nfree = 0;
            for (uint64_t x = lo[k]; x < lo[k] + caps[k]; ++x)
                if (!(taken[x >> 6] & (1ull << (x & 63)))) freelist[nfree++] = (uint32_t)x;
            const uint64_t take = want < nfree ? want : nfree;
            for (uint64_t i = 0; i < take; ++i) {
                const uint64_t j = i + sm64_next(&s) % (nfree - i);
                const uint32_t t = freelist[i];
                freelist[i] = freelist[j];
                freelist[j] = t;
                taken[freelist[i] >> 6] |= 1ull << (freelist[i] & 63);
                tmp[filled++] = freelist[i];
            }
            carry = want - take;
        }
        if (filled != n) {
            rc = -3;
            goto done;
        }
    }
    {
        feistel_t f;
        feistel_init(&f, n, sm64_next(&s));
        perm_ctx c = {&f, out, tmp};
        parallel_for(n, perm_range, &c);
    }
done:
    free(lo);
    free(caps);
    free(sizes);
    free(taken);
    free(freelist);
    free(tmp);
    return rc;
}
