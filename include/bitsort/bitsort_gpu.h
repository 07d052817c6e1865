#ifndef BITSORT_BITSORT_GPU_H
#define BITSORT_BITSORT_GPU_H

/*
 * Additive B200 extensions to the bitsort C ABI (SURVEY.md §8(b) "Extensions").
 * None of these exist in the reference; they sit beside bws_sort
 * (proj/include/bitsort/bitsort.h:89-90) without changing it, so an unmodified
 * reference caller never sees them. All pointers are plain device or host
 * addresses; `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream). Every function returns bws_status and sets bws_last_error() exactly
 * like the reference entry points (capi.cpp:19-41).
 *
 * Keys are uint32, distinct, in [0, key_range). key_range is a power of two or
 * any value in [1, 2^32]; 0 means "derive from the data" (max key + 1).
 */

#include "bitsort.h"

#ifdef __cplusplus
extern "C" {
#endif

/* bws_sort(data, count, 32, 1, BWS_ALG_BITWISE) with a key-range hint: skips
 * the max-reduction pass. Keys >= key_range -> BWS_ERROR_DATA, data untouched. */
BITSORT_API bws_status bws_sort_u32_range(void* data, size_t count, uint64_t key_range);

/* Device-resident sort, stream-ordered, no host synchronisation (also with
 * key_range == 0: the range is then derived on the device by the direct
 * pipeline, which is slower for large inputs than giving the hint), so it can
 * be captured in a CUDA graph. `keys` and `out` are device pointers (they may
 * alias for an in-place sort). On return the work is queued on `stream`;
 * bws_gpu_sort_check() synchronises and validates the most recent async sort
 * on this device — other library calls in between do not disturb its result
 * (its control block is set aside first). */
BITSORT_API bws_status bws_gpu_sort_device_async(const uint32_t* keys, size_t count,
                                                 uint32_t* out, uint64_t key_range,
                                                 void* stream);

/* bws_gpu_sort_device_async for keys in [key_lo, key_lo + key_range)
 * (key_lo + key_range <= 2^32): the bucketed pipeline works on key - key_lo,
 * so a rank's slice of a larger range (multi-GPU key all-to-all) costs no
 * more than a sort starting at 0. Checked by bws_gpu_sort_check. */
BITSORT_API bws_status bws_gpu_sort_range_device_async(const uint32_t* keys, size_t count,
                                                       uint32_t* out, uint32_t key_lo,
                                                       uint64_t key_range, void* stream);

/* Range split for the multi-GPU key all-to-all: writes
 * the `count` device keys (all < key_range) to `out` grouped by part, part p
 * holding keys in [p * W, (p + 1) * W) ∩ [0, key_range), in part order (order
 * inside a part is unspecified), and the number of keys of each part to the
 * device array d_counts[parts] (uint32). *part_width receives W (the smallest
 * q * 2^s >= ceil(key_range / parts), q <= 8). Synchronises `stream`; keys >=
 * key_range -> BWS_ERROR_DATA. */
BITSORT_API bws_status bws_gpu_range_split(const uint32_t* keys, size_t count, uint64_t key_range,
                                           int parts, uint32_t* out, uint32_t* d_counts,
                                           uint64_t* part_width, void* stream);

/* Synchronises `stream` (and the sort's own stream) and validates the most
 * recent bws_gpu_sort_(range_)device_async on the current device:
 * BWS_ERROR_DATA on duplicates / out-of-range keys.
 * *distinct_out (optional) receives the number of keys written. */
BITSORT_API bws_status bws_gpu_sort_check(void* stream, uint64_t* distinct_out);

/* Per-rank building blocks for the multi-GPU path (one process per GPU).
 *   bitset_build: the full bitset of `count` keys (device) in [0, key_range)
 *                 at `bits` (ceil(key_range/32) uint32 words, overwritten;
 *                 no prior clearing needed). Large inputs go through the
 *                 bucketed SMEM-staged build (no global atomics), small ones
 *                 through K1 clear + K2 scatter.
 *   bitset_scan:  K3 over n_words words at `bits` (a rank's slice), writing
 *                 key_base + bit_index for every set bit, ascending, to `out`
 *                 (capacity out_capacity keys). The number of keys is written
 *                 to the device uint64 at `d_total`. */
BITSORT_API bws_status bws_gpu_bitset_build(const uint32_t* keys, size_t count, uint32_t* bits,
                                            uint64_t key_range, void* stream);
BITSORT_API bws_status bws_gpu_bitset_scan(const uint32_t* bits, uint64_t n_words,
                                           uint32_t key_base, uint32_t* out,
                                           uint64_t out_capacity, uint64_t* d_total,
                                           void* stream);

/* Peer-to-peer replacement of the reduce-scatter (one process per GPU on an
 * NVLink/NVSwitch node): every rank exports its full bitset with
 * bws_gpu_ipc_get_handle, opens the peers' with bws_gpu_ipc_open, and after a
 * cross-rank barrier ORs the words of its own slice from all nsrc (<= 8)
 * bitsets into `dst` with bws_gpu_bitset_or_gather (`srcs` is a host array of
 * device pointers, each already offset to the slice; peer pointers read over
 * NVLink). OR equals the SUM of the reduce-scatter on distinct keys and loses
 * bits on duplicates, which the popcount total then reports. */
#define BWS_GPU_IPC_HANDLE_BYTES 64
BITSORT_API bws_status bws_gpu_bitset_or_gather(const uint32_t* const* srcs, int nsrc, uint64_t n_words,
                                                uint32_t* dst, void* stream);
/* The exchange fused into the scan: bws_gpu_bitset_scan over the virtual
 * slice OR_s srcs[s][0, n_words) (srcs[0] the local bitset's slice, the rest
 * peers' slices opened through CUDA IPC). One kernel: every scan tile ORs the
 * peers' words (16-byte loads over NVLink/NVSwitch) into its shared-memory
 * copy of the local words, so no gathered slice is written to HBM and read
 * back. Same outputs and d_total as bws_gpu_bitset_or_gather followed by
 * bws_gpu_bitset_scan. Sources not 16-byte aligned take exactly that
 * two-kernel route. */
BITSORT_API bws_status bws_gpu_bitset_scan_sources(const uint32_t* const* srcs, int nsrc,
                                                   uint64_t n_words, uint32_t key_base,
                                                   uint32_t* out, uint64_t out_capacity,
                                                   uint64_t* d_total, void* stream);
/* The exchange fused into the build (push variant): builds the bitset of
 * `count` keys in [0, key_range) bucket by bucket in shared memory and ORs
 * each finished bucket straight into the owner's slice with bulk
 * OR-reductions: slices[r] (device pointer, local or a peer's opened through
 * CUDA IPC, 16-byte aligned, zeroed by its owner beforehand) holds words
 * [r * slice_words, (r + 1) * slice_words) of the global bitset; slice_words
 * a multiple of 4 and nslices * slice_words >= ceil(key_range / 32). Every
 * rank pushes into every slice; after a cross-rank barrier each owner scans
 * its slice with bws_gpu_bitset_scan. No full bitset is materialised on any
 * rank and no separate collective runs. */
BITSORT_API bws_status bws_gpu_bitset_push(const uint32_t* keys, size_t count, uint64_t key_range,
                                           uint32_t* const* slices, int nslices, uint64_t slice_words,
                                           void* stream);
/* handle_out: BWS_GPU_IPC_HANDLE_BYTES bytes naming dev_ptr's allocation;
 * *offset_out: dev_ptr's byte offset in it (add it to the pointer
 * bws_gpu_ipc_open returns in the peer process). */
BITSORT_API bws_status bws_gpu_ipc_get_handle(const void* dev_ptr, void* handle_out, uint64_t* offset_out);
BITSORT_API bws_status bws_gpu_ipc_open(const void* handle, void** dev_ptr_out);
BITSORT_API bws_status bws_gpu_ipc_close(void* dev_ptr);

/* Scatter-kernel staging switches (tests / ablations; default BWS_SCATTER_AUTO). */
typedef enum bws_scatter_mode {
    BWS_SCATTER_AUTO = 0,      /* per tile: SMEM staging if the tile's span fits, else
                                  warp-aggregated (match.any) when a warp's span is
                                  narrow, else plain atomicOr */
    BWS_SCATTER_PLAIN = 1,     /* one atomicOr per key */
    BWS_SCATTER_WARP_AGG = 2,  /* always warp-aggregate */
    BWS_SCATTER_SMEM = 3       /* SMEM staging when the span fits, else warp-aggregate */
} bws_scatter_mode;
BITSORT_API bws_status bws_gpu_set_scatter_mode(bws_scatter_mode mode);

/* Sort pipeline for bws_sort / bws_sort_u32_range / bws_gpu_sort_device_async
 * (default BWS_PATH_AUTO, or env BITSORT_PATH=auto|direct|bucketed|fused|fused_direct|small).
 *   DIRECT   : K2 global-bitset scatter + K3 decoupled-lookback scan
 *   BUCKETED : key-range bucketing (coalesced) + per-bucket SMEM bitset +
 *              fused extraction; no global bitset
 *   FUSED    : one persistent kernel; the bitset of a pass split into per-SM
 *              shared-memory slices, keys routed to their slice's SM through
 *              L2-resident rings (key ranges up to ~2^28 on a 148-SM B200;
 *              larger ranges take BUCKETED)
 *   FUSED_DIRECT : one persistent kernel: keys ORed into the global bitset
 *              (L2-resident), a grid barrier, then every SM counts and
 *              extracts its slice in shared memory (small sorts)
 *   SMALL    : one cooperative launch for small sorts with a range hint: keys
 *              ORed into the global bitset, a grid barrier, every SM counts
 *              its slice in registers, tagged count exchange, extraction
 *              straight from registers (ranges up to 2^27 on a 148-SM B200)
 *   AUTO     : BUCKETED for n >= 2^21; below, SMALL when a range hint of at
 *              most 2^25 is given, else DIRECT */
typedef enum bws_path {
    BWS_PATH_AUTO = 0,
    BWS_PATH_DIRECT = 1,
    BWS_PATH_BUCKETED = 2,
    BWS_PATH_FUSED = 3,
    BWS_PATH_FUSED_DIRECT = 4,
    BWS_PATH_SMALL = 5
} bws_path;
BITSORT_API bws_status bws_gpu_set_path(bws_path path);


/* Number of kernels this library has launched in this process (evidence for
 * bench.py's gpu_launches). */
BITSORT_API uint64_t bws_gpu_launch_count(void);

/* Per-kernel CUDA-event timing for bench.py's live roofline. While enabled,
 * every kernel this library launches is bracketed by events on its stream.
 * bws_gpu_kernel_timings() synchronises those events and writes one line per
 * kernel, "<name> <launches> <total_ms>\n", for the launches since the
 * previous call. */
BITSORT_API bws_status bws_gpu_set_kernel_timing(int enable);
BITSORT_API bws_status bws_gpu_kernel_timings(char* buf, size_t buf_size);

/* Multi-GPU bws_sort in one process: with G > 1 devices,
 * bws_sort / bws_sort_u32_range on a HOST array of unsigned 32-bit keys
 * (>= 2^20 keys, env BITSORT_MULTI_MIN_KEYS) shards the array over the G
 * devices (each shard over its own PCIe link), builds a full bitset per
 * device, combines them (NCCL reduce-scatter with ncclSum on uint32 words when
 * the devices are distinct and libnccl.so.2 loads, else — or with env
 * BITSORT_EXCHANGE=p2p — a fused scan reading every device's bitset slice over
 * peer access), scans one key-range slice per device and writes every slice
 * back at its offset. Repeated keys take the single-GPU counting pass. Other
 * widths, signed keys and device arrays run on one GPU.
 *   bws_gpu_set_device_count(G): devices 0 .. G-1 (1 = single GPU; default:
 *       env BITSORT_GPUS, else 1);
 *   bws_gpu_set_devices(list, G): an explicit list (env BITSORT_DEVICES,
 *       e.g. "0,1,2,3"); a device may appear more than once (logical ranks
 *       sharing a GPU: the P2P exchange; used by the tests on one GPU);
 *   bws_gpu_device_count(): the current G.
 * At most 8 logical ranks. BWS_ERROR_CONFIG for an invisible device. */
BITSORT_API bws_status bws_gpu_set_device_count(int count);
BITSORT_API bws_status bws_gpu_set_devices(const int* devices, int count);
BITSORT_API int bws_gpu_device_count(void);

/* Releases cached device buffers, streams and communicators. */
BITSORT_API void bws_gpu_shutdown(void);

#ifdef __cplusplus
}
#endif

#endif /* BITSORT_BITSORT_GPU_H */
