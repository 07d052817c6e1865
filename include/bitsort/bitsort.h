#ifndef BITSORT_BITSORT_H
#define BITSORT_BITSORT_H

/*
 * bitsort C ABI — B200 build (drop-in for the reference's sort surface).
 *
 * Every declaration below keeps the reference's name, value and signature so a
 * caller compiled against /root/reference/proj/include/bitsort/bitsort.h links
 * against this libbitsort.so.1 unchanged:
 *
 *   bws_status      enum   <- proj/include/bitsort/bitsort.h:29-36
 *   bws_algorithm   enum   <- proj/include/bitsort/bitsort.h:38-45
 *   bws_version            <- proj/include/bitsort/bitsort.h:47   (impl capi.cpp:96)
 *   bws_last_error         <- proj/include/bitsort/bitsort.h:49-52 (impl capi.cpp:98)
 *   bws_algorithm_name     <- proj/include/bitsort/bitsort.h:83   (impl capi.cpp:164-174)
 *   bws_algorithm_from_name<- proj/include/bitsort/bitsort.h:84   (impl capi.cpp:176-184)
 *   bws_sort               <- proj/include/bitsort/bitsort.h:86-90 (impl capi.cpp:186-197)
 *
 * The reference's bit-utility (bitsort.h:54-79), trace (:92-99) and benchmark
 * handle (:101-143) entry points are not on the sort path and are not part of
 * this library.
 *
 * Domain of the GPU bws_sort: every algorithm id (a sort's output is unique, so
 * BITWISE, BITWISE_SKIP_EMPTY, INSERTION, MERGE, COUNTING and PLATFORM all run
 * the GPU pipelines below; COUNTING keeps the reference's span limit: max - min
 * >= 2^26 is BWS_ERROR_RANGE, baselines.hpp:95-110), unsigned or signed keys
 * (mapped onto the unsigned order by flipping the sign bit on load and store),
 * naturally aligned:
 *   width 32  the bitset sort (the hot path); repeated keys are detected and
 *             sorted by a GPU counting-sort pass, as the reference sorts them;
 *   width 8/16  a GPU counting sort over the type's range;
 *   width 64  keys whose span max - min is below 2^32 narrowed to the 32-bit
 *             path; wider spans by a stable LSD radix sort (8-bit digits).
 * There is no CPU fallback: without a CUDA device every call that sorts
 * returns BWS_ERROR_INTERNAL.
 * Additive GPU extensions live in bitsort_gpu.h.
 */

#include <stddef.h>
#include <stdint.h>

#if defined(_WIN32)
#if defined(BITSORT_BUILD)
#define BITSORT_API __declspec(dllexport)
#else
#define BITSORT_API __declspec(dllimport)
#endif
#else
#define BITSORT_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum bws_status {
    BWS_OK = 0,
    BWS_ERROR_CONFIG = 1,    /* unsupported width/signedness/algorithm, bad API usage */
    BWS_ERROR_DATA = 2,      /* null data, duplicate keys, key outside the range hint */
    BWS_ERROR_INTEGRITY = 3, /* kept for ABI value parity; not produced by bws_sort */
    BWS_ERROR_RANGE = 4,     /* range hint out of bounds; COUNTING key span >= 2^26 */
    BWS_ERROR_INTERNAL = 5   /* CUDA / NCCL failure (message in bws_last_error) */
} bws_status;

typedef enum bws_algorithm {
    BWS_ALG_BITWISE = 0,
    BWS_ALG_BITWISE_SKIP_EMPTY = 1,
    BWS_ALG_INSERTION = 2,
    BWS_ALG_MERGE = 3,
    BWS_ALG_COUNTING = 4,
    BWS_ALG_PLATFORM = 5
} bws_algorithm;

/* "1.0.0", the reference's library version (capi.cpp:96). */
BITSORT_API const char* bws_version(void);

/* Message of the most recent failing call on this thread; "" after a call
 * that succeeded. Valid until the next call on the same thread. */
BITSORT_API const char* bws_last_error(void);

BITSORT_API const char* bws_algorithm_name(bws_algorithm algorithm);
BITSORT_API bws_status bws_algorithm_from_name(const char* name, bws_algorithm* out);

/* In-place ascending sort of `count` elements at `data`.
 * `data` may be host memory (pageable or pinned) or CUDA device memory. */
BITSORT_API bws_status bws_sort(void* data, size_t count, uint32_t width, int is_unsigned,
                                bws_algorithm algorithm);

#ifdef __cplusplus
}
#endif

#endif /* BITSORT_BITSORT_H */
