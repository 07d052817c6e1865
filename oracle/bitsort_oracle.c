/*
 * CPU ORACLE — test infrastructure only. Nothing in the product path
 * (paper_1312_0138_b200/, libbitsort.so) links, loads or calls this file; it is
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs as the checker.
 *
 * Plain-C restatement of the reference's sort for unsigned keys:
 *
 *   oracle_bitwise_sort_u{8,16,32,64}
 *     <- bws::detail::partition_pass        proj/src/bitsort.hpp:84-103
 *        (stable split on bit k: zeros bucket, ones bucket, copy back zeros
 *        then ones)
 *     <- bws::detail::sort_same_sign_impl   proj/src/bitsort.hpp:111-129
 *        (one pass per bit, k = 0..t-1; optional OR-fold skip of empty bits
 *        :117-123)
 *     <- bws::detail::bitwise_sort_impl     proj/src/bitsort.hpp:131-136
 *        (unsigned: no sign split)
 *     pass_count<unsigned T> = t            proj/src/bitsort.hpp:46-47
 *
 *   oracle_bitwise_sort_s{8,16,32,64}
 *     <- bws::detail::bitwise_sort_impl     proj/src/bitsort.hpp:137-151
 *        (signed: stable split into negatives and non-negatives, each group
 *        sorted by the same-sign passes on its two's-complement bits, then
 *        negatives written back first)
 *     pass_count<signed T> = t - 1          proj/src/bitsort.hpp:46-47
 *        (the sign bit is constant inside a group and never inspected)
 *
 *   oracle_splitmix64_next / oracle_generate_uniform_u32
 *     <- bws::splitmix64                    proj/src/generator.hpp:21-30
 *     <- bws::mix64                         proj/src/generator.hpp:32-36
 *     <- bws::generate_input<uint32_t>(n, uniform_full_range, seed, trial)
 *                                           proj/src/generator.hpp:91-103
 *
 *   oracle_bitset_build / oracle_bitset_scan
 *     The north-star algorithm restated on the CPU for checking the multi-rank
 *     host logic: bws::counting_sort (proj/src/baselines.hpp:99-122) with 1-bit
 *     counters, valid because keys are distinct.
 *
 * Pinned against the reference: tests/test_oracle.py compares these functions
 * with tests/golden/ fixtures produced by the reference's own bws_sort
 * (tests/golden/gen_golden.cpp) and with oracle/_ref/libbitsort_ref.so when it
 * is present.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_API __attribute__((visibility("default")))

/* One stable partition pass on bit k followed by the copy-back
 * (bitsort.hpp:88-98). */
#define DEFINE_BITWISE_SORT(SUFFIX, T, BITS)                                             \
    ORACLE_API int oracle_bitwise_sort_##SUFFIX(T* a, size_t n, int skip_empty_bits) {   \
        if (n == 0) return 0;                                                            \
        T* zeros = (T*)calloc(n, sizeof(T));                                             \
        T* ones = (T*)calloc(n, sizeof(T));                                              \
        if (!zeros || !ones) {                                                           \
            free(zeros);                                                                 \
            free(ones);                                                                  \
            return -1;                                                                   \
        }                                                                                \
        T set_bits = (T)~(T)0;                                                           \
        if (skip_empty_bits) {                                                           \
            set_bits = 0;                                                                \
            for (size_t i = 0; i < n; ++i) set_bits |= a[i];                             \
        }                                                                                \
        for (unsigned k = 0; k < (BITS); ++k) {                                          \
            if (skip_empty_bits && ((set_bits >> k) & 1u) == 0) continue;                \
            size_t zc = 0, oc = 0;                                                       \
            for (size_t i = 0; i < n; ++i) {                                             \
                if ((a[i] >> k) & 1u)                                                    \
                    ones[oc++] = a[i];                                                   \
                else                                                                     \
                    zeros[zc++] = a[i];                                                  \
            }                                                                            \
            size_t j = 0;                                                                \
            for (size_t z = 0; z < zc; ++z) a[j++] = zeros[z];                           \
            for (size_t o = 0; o < oc; ++o) a[j++] = ones[o];                            \
        }                                                                                \
        free(zeros);                                                                     \
        free(ones);                                                                      \
        return 0;                                                                        \
    }

DEFINE_BITWISE_SORT(u8, uint8_t, 8)
DEFINE_BITWISE_SORT(u16, uint16_t, 16)
DEFINE_BITWISE_SORT(u32, uint32_t, 32)
DEFINE_BITWISE_SORT(u64, uint64_t, 64)

/* Same-sign passes over bits 0 .. BITS-2 of the unsigned patterns (the sign
 * split already made the top bit constant), reusing the unsigned routine's
 * pass on a group (bitsort.hpp:111-129 with pass_count = t - 1). */
#define DEFINE_SIGNED_SORT(SUFFIX, ST, UT, BITS)                                          \
    static void same_sign_##SUFFIX(UT* g, size_t n, UT* zeros, UT* ones, int skip) {       \
        UT set_bits = (UT)~(UT)0;                                                          \
        if (skip) {                                                                        \
            set_bits = 0;                                                                  \
            for (size_t i = 0; i < n; ++i) set_bits |= g[i];                               \
        }                                                                                  \
        for (unsigned k = 0; k + 1 < (BITS); ++k) {                                        \
            if (skip && ((set_bits >> k) & 1u) == 0) continue;                             \
            size_t zc = 0, oc = 0;                                                         \
            for (size_t i = 0; i < n; ++i) {                                               \
                if ((g[i] >> k) & 1u)                                                      \
                    ones[oc++] = g[i];                                                     \
                else                                                                       \
                    zeros[zc++] = g[i];                                                    \
            }                                                                              \
            size_t j = 0;                                                                  \
            for (size_t z = 0; z < zc; ++z) g[j++] = zeros[z];                             \
            for (size_t o = 0; o < oc; ++o) g[j++] = ones[o];                              \
        }                                                                                  \
    }                                                                                      \
    ORACLE_API int oracle_bitwise_sort_##SUFFIX(ST* a, size_t n, int skip_empty_bits) {    \
        if (n == 0) return 0;                                                              \
        UT* neg = (UT*)calloc(n, sizeof(UT));                                              \
        UT* pos = (UT*)calloc(n, sizeof(UT));                                              \
        UT* zeros = (UT*)calloc(n, sizeof(UT));                                            \
        UT* ones = (UT*)calloc(n, sizeof(UT));                                             \
        if (!neg || !pos || !zeros || !ones) {                                             \
            free(neg);                                                                     \
            free(pos);                                                                     \
            free(zeros);                                                                   \
            free(ones);                                                                    \
            return -1;                                                                     \
        }                                                                                  \
        size_t nn = 0, np = 0;                                                             \
        for (size_t i = 0; i < n; ++i) {                                                   \
            if (a[i] < 0)                                                                  \
                neg[nn++] = (UT)a[i];                                                      \
            else                                                                           \
                pos[np++] = (UT)a[i];                                                      \
        }                                                                                  \
        same_sign_##SUFFIX(neg, nn, zeros, ones, skip_empty_bits);                         \
        same_sign_##SUFFIX(pos, np, zeros, ones, skip_empty_bits);                         \
        size_t j = 0;                                                                      \
        for (size_t i = 0; i < nn; ++i) a[j++] = (ST)neg[i];                               \
        for (size_t i = 0; i < np; ++i) a[j++] = (ST)pos[i];                               \
        free(neg);                                                                         \
        free(pos);                                                                         \
        free(zeros);                                                                       \
        free(ones);                                                                        \
        return 0;                                                                          \
    }

DEFINE_SIGNED_SORT(s8, int8_t, uint8_t, 8)
DEFINE_SIGNED_SORT(s16, int16_t, uint16_t, 16)
DEFINE_SIGNED_SORT(s32, int32_t, uint32_t, 32)
DEFINE_SIGNED_SORT(s64, int64_t, uint64_t, 64)

/* splitmix64 step (generator.hpp:24-29). `state` is advanced in place. */
ORACLE_API uint64_t oracle_splitmix64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* mix64(h, v) = splitmix64{h ^ v}.next() (generator.hpp:32-36). */
ORACLE_API uint64_t oracle_mix64(uint64_t h, uint64_t v) {
    uint64_t s = h ^ v;
    return oracle_splitmix64_next(&s);
}

/* generate_input<uint32_t>(n, uniform_full_range, seed, trial): the stream seed
 * is mix64(mix64(mix64(seed, 32), n), trial) and each element is the low 32
 * bits of one splitmix64 draw (generator.hpp:95, :101-103). */
ORACLE_API void oracle_generate_uniform_u32(uint32_t* out, size_t n, uint64_t seed,
                                            uint32_t trial) {
    uint64_t state = oracle_mix64(oracle_mix64(oracle_mix64(seed, 32), (uint64_t)n), trial);
    for (size_t i = 0; i < n; ++i) out[i] = (uint32_t)oracle_splitmix64_next(&state);
}

/* FNV-1a 64 over a byte range (fixture checksums). */
ORACLE_API uint64_t oracle_fnv1a64(const void* data, size_t bytes) {
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < bytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* Sets bit (x & 31) of word (x >> 5) for every key < key_range in a zeroed
 * ceil(key_range/32)-word bitset. Returns the number of keys outside the range. */
ORACLE_API uint64_t oracle_bitset_build(const uint32_t* keys, size_t n, uint32_t* bits,
                                        uint64_t key_range) {
    const uint64_t words = (key_range + 31) / 32;
    memset(bits, 0, words * sizeof(uint32_t));
    uint64_t bad = 0;
    for (size_t i = 0; i < n; ++i) {
        if ((uint64_t)keys[i] >= key_range) {
            ++bad;
            continue;
        }
        bits[keys[i] >> 5] |= 1u << (keys[i] & 31);
    }
    return bad;
}

/* Emits key_base + bit index of every set bit of n_words words, ascending, to
 * out (at most out_capacity keys). Returns the number of set bits. */
ORACLE_API uint64_t oracle_bitset_scan(const uint32_t* bits, uint64_t n_words, uint32_t key_base,
                                       uint32_t* out, uint64_t out_capacity) {
    uint64_t count = 0;
    for (uint64_t w = 0; w < n_words; ++w) {
        uint32_t x = bits[w];
        while (x) {
            const unsigned b = (unsigned)__builtin_ctz(x);
            x &= x - 1;
            if (count < out_capacity) out[count] = key_base + (uint32_t)(w * 32u + b);
            ++count;
        }
    }
    return count;
}
