// Internal host-side interface of libbitsort.so shared by capi.cpp (the C
// ABI, single-GPU orchestration) and multi.cpp (single-process multi-GPU
// orchestration). Nothing here is exported (the library is built with
// -fvisibility=hidden and a version script that exports only bws_*).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges are no-ops unless a tool attaches

#include "bitsort/bitsort.h"
#include "bitsort/bitsort_gpu.h"
#include "kernels.h"

namespace bws_host {

// NVTX range over a host-side phase (enqueue of a pipeline, staging copies,
// entry points), visible in nsys / ncu timelines as "bitsort:<name>".
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};


using bws_gpu::Ctrl;

struct config_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct data_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct internal_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t err, const char* what) {
    if (err != cudaSuccess)
        throw internal_error(std::string(what) + ": " + cudaGetErrorName(err) + " (" +
                             cudaGetErrorString(err) + ")");
}

constexpr uint64_t kMaxKeyRange = 1ull << 32;
constexpr uint64_t kMaxWords = kMaxKeyRange / 32;               // 2^27 words = 512 MiB
constexpr size_t kMaxTiles = (kMaxWords + bws_gpu::SCAN_TILE_WORDS - 1) / bws_gpu::SCAN_TILE_WORDS;
// Ctrl + tile status (v1: 8 B per 2048-word tile; the two-pass v2 scan keeps
// offsets, tile counts and 16 segment counts per 8192-word tile there)
constexpr size_t kCtrlBytes = sizeof(Ctrl) + 4 * kMaxTiles * sizeof(unsigned long long);

extern std::atomic<uint64_t> g_launches;
extern std::atomic<int> g_scatter_mode;
constexpr size_t kBucketedMinKeys = size_t(1) << 21;
constexpr size_t kSmallMaxRange = size_t(1) << 25;    // AUTO: KS for hinted sorts below kBucketedMinKeys keys
                                                       // whose range is at most this (2 bitset vectors per thread;
                                                       // at 7 per thread, M = 2^27, KS measured no faster than K2 + K3)
constexpr size_t kFusedMinKeys = size_t(1) << 16;        // AUTO: KD from here ...
constexpr size_t kFusedDirectMaxKeys = 0;  // ... up to here (0: AUTO never takes KD: a tie with K2+K3 on C1)

int current_path();

constexpr size_t kStageChunk = size_t(16) << 20;  // bytes per pinned bounce buffer

struct DeviceCtx {
    std::mutex mu;
    bool ready = false;
    int device = -1;
    bws_gpu::LaunchGeometry geo;
    cudaStream_t stream = nullptr;
    uint32_t* bits = nullptr;  // kMaxWords words; all-zero between sorts unless bits_dirty
    bool bits_dirty = true;
    unsigned char* ctrl_mem = nullptr;  // Ctrl followed by the K3 tile-status array
    Ctrl* host_ctrl = nullptr;          // pinned landing buffer of the control block read-back
    uint32_t* keys = nullptr;           // staging for host arrays
    size_t keys_cap = 0;
    uint32_t* parted = nullptr;         // bucketed path: keys grouped by bucket
    size_t parted_cap = 0;
    void* bucket_scratch = nullptr;     // bucketed path: histograms, totals, bases
    void* wide = nullptr;               // staging for host arrays of 8/16/64-bit keys
    size_t wide_cap = 0;
    void* width_scratch = nullptr;      // 8/16-bit histogram + prefix, 64-bit min/max
    void* fused = nullptr;              // KF ring state (persistent; re-initialised after a fault)
    bool fused_dirty = true;
    void* small = nullptr;              // KS arrival counter + tagged counts (zeroed once)
    bool small_dirty = true;            // zero the KS state before the next launch (first use, fault)
    uint32_t* fused_saved = nullptr;    // KF pass-0 slices
    size_t fused_saved_words = 0;
    // the most recent bws_gpu_sort_(range_)device_async on this device, checked
    // by bws_gpu_sort_check; once another library call reuses the control
    // block its final state is first copied (stream-ordered) to snap()
    struct AsyncSort {
        bool active = false;
        cudaStream_t stream = nullptr;
        size_t count = 0;
        uint64_t range = 0;  // 0 = derived
        bool snapped = false;
    } pending;
    // key range the next in-place bws_sort of a device array without a hint is
    // planned for (0: none yet, K0 derives it): the range the previous such
    // sort's keys really had, rounded up — see sort_u32
    uint64_t spec_range = 0;
    int spec_misses = 0;      // consecutive sorts whose keys outgrew spec_range
    int spec_cooldown = 0;    // sorts left that run K0 without speculating (after two misses in a row)
    uint64_t spec_small = 0;  // likewise for unhinted sorts below 2^21 keys (KS instead of K2 + K3)
    void* bounce[2] = {nullptr, nullptr};  // pinned staging for pageable host arrays
    cudaEvent_t bounce_ev[2] = {nullptr, nullptr};
    cudaEvent_t done = nullptr;   // recorded after every queued sort: orders the
                                  // shared bitset/control block across streams

    Ctrl* ctrl() { return reinterpret_cast<Ctrl*>(ctrl_mem); }
    Ctrl* snap() { return reinterpret_cast<Ctrl*>(ctrl_mem + kCtrlBytes); }
    unsigned long long* status() {
        return reinterpret_cast<unsigned long long*>(ctrl_mem + sizeof(Ctrl));
    }

    void init(int dev) {
        if (ready) return;
        device = dev;
        cuda_check(cudaSetDevice(dev), "cudaSetDevice");
        cuda_check(bws_gpu::query_geometry(dev, &geo), "occupancy query");
        cuda_check(bws_gpu::configure_bucket_kernels(dev, &geo), "bucket kernel configuration");
        cuda_check(bws_gpu::configure_scan2(dev, &geo), "scan kernel configuration");
        cuda_check(bws_gpu::configure_width_kernels(dev, &geo), "width kernel configuration");
        cuda_check(bws_gpu::configure_fused(dev, &geo), "fused kernel configuration");
        cuda_check(bws_gpu::configure_small(dev, &geo), "small-sort kernel configuration");
        cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaMalloc(&ctrl_mem, kCtrlBytes + sizeof(Ctrl)), "cudaMalloc(control block)");
        cuda_check(cudaHostAlloc(&host_ctrl, sizeof(Ctrl), cudaHostAllocDefault), "cudaHostAlloc(control block)");
        pending = AsyncSort{};
        cuda_check(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "cudaEventCreate");
        bws_gpu::BucketPlan widest;
        widest.nb = bws_gpu::MAX_BUCKETS;
        const int max_shares = geo.part_blocks > geo.part_blocks_narrow ? geo.part_blocks : geo.part_blocks_narrow;
        const size_t scratch_bytes = bws_gpu::bucket_scratch_bytes(widest, max_shares) + 64;
        cuda_check(cudaMalloc(&bucket_scratch, scratch_bytes), "cudaMalloc(bucket scratch)");
        // the slab fill counters must start at zero (KB3 re-zeroes them after each sort)
        cuda_check(cudaMemset(bucket_scratch, 0, scratch_bytes), "bucket scratch clear");
        bits_dirty = true;
        ready = true;
    }

    // The direct path's 2^32-bit bitset (512 MiB), allocated on its first use
    // (bucketed sorts never need it).
    void ensure_bits() {
        if (bits) return;
        cuda_check(cudaMalloc(&bits, kMaxWords * sizeof(uint32_t)), "cudaMalloc(bitset 512 MiB)");
        bits_dirty = true;
    }

    void ensure_keys(size_t n) {
        if (n <= keys_cap) return;
        if (keys) cuda_check(cudaFree(keys), "cudaFree(keys)");
        keys = nullptr;
        keys_cap = 0;
        const size_t cap = n + n / 4;
        cuda_check(cudaMalloc(&keys, cap * sizeof(uint32_t)), "cudaMalloc(key staging)");
        keys_cap = cap;
    }

    // Bucket buffer for n keys under `plan`: the slab layout's slots when it
    // applies (bws_gpu::slab_slots), else n. Returns the usable capacity.
    size_t ensure_parted(size_t n, const bws_gpu::BucketPlan& plan) {
        size_t need = static_cast<size_t>(bws_gpu::slab_slots(plan, n)) > n
                          ? static_cast<size_t>(bws_gpu::slab_slots(plan, n))
                          : n;
        if (static_cast<size_t>(bws_gpu::chunk_slots(plan, n)) > need)
            need = static_cast<size_t>(bws_gpu::chunk_slots(plan, n));
        if (need <= parted_cap) return parted_cap;
        if (parted) cuda_check(cudaFree(parted), "cudaFree(parted)");
        parted = nullptr;
        parted_cap = 0;
        const size_t cap = need + n / 8 + 64;  // KB4 bulk copies may read up to 12 bytes past a bucket
        if (cudaMalloc(&parted, cap * sizeof(uint32_t)) != cudaSuccess) {
            // the slab is an optimisation: fall back to the packed layout's n slots
            cudaGetLastError();
            const size_t packed = n + n / 8 + 64;
            cuda_check(cudaMalloc(&parted, packed * sizeof(uint32_t)), "cudaMalloc(bucket keys)");
            parted_cap = packed - 64;
            return parted_cap;
        }
        parted_cap = cap - 64;
        return parted_cap;
    }

    void* ensure_wide(size_t bytes) {
        if (bytes > wide_cap) {
            if (wide) cuda_check(cudaFree(wide), "cudaFree(wide keys)");
            wide = nullptr;
            wide_cap = 0;
            cuda_check(cudaMalloc(&wide, bytes), "cudaMalloc(wide keys)");
            wide_cap = bytes;
        }
        if (!width_scratch)
            cuda_check(cudaMalloc(&width_scratch, bws_gpu::width_scratch_bytes()), "cudaMalloc(width scratch)");
        return wide;
    }

    // KF state (rings, counters) and the pass-0 slice buffer for `plan`.
    void ensure_fused(const bws_gpu::FusedPlan& plan, cudaStream_t s) {
        if (!fused) {
            cuda_check(cudaMalloc(&fused, bws_gpu::fused_state_bytes(plan.G)), "cudaMalloc(fused rings)");
            fused_dirty = true;
        }
        if (fused_dirty) {
            cuda_check(bws_gpu::init_fused_state(fused, plan.G, s), "fused ring init");
            fused_dirty = false;
        }
        const size_t words = plan.P == 2 ? static_cast<size_t>(plan.G) * (plan.S / 32) : 0;
        if (words > fused_saved_words) {
            if (fused_saved) cuda_check(cudaFree(fused_saved), "cudaFree(fused slices)");
            fused_saved = nullptr;
            fused_saved_words = 0;
            cuda_check(cudaMalloc(&fused_saved, words * sizeof(uint32_t)), "cudaMalloc(fused slices)");
            fused_saved_words = words;
        }
    }

    // KS state (arrival counter + slice histograms), zeroed on first use and after a fault.
    void ensure_small(cudaStream_t s) {
        if (!small) {
            cuda_check(cudaMalloc(&small, bws_gpu::small_state_bytes()), "cudaMalloc(small-sort state)");
            small_dirty = true;
        }
        if (small_dirty) {
            cuda_check(cudaMemsetAsync(small, 0, bws_gpu::small_state_bytes(), s), "small-sort state reset");
            small_dirty = false;
        }
    }

    void ensure_bounce() {
        if (bounce[0]) return;
        for (int i = 0; i < 2; ++i) {
            cuda_check(cudaHostAlloc(&bounce[i], kStageChunk, cudaHostAllocDefault), "cudaHostAlloc(staging)");
            cuda_check(cudaEventCreateWithFlags(&bounce_ev[i], cudaEventDisableTiming), "cudaEventCreate");
        }
    }

    void release() {
        if (!ready) return;
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        for (int i = 0; i < 2; ++i) {
            if (bounce[i]) cudaFreeHost(bounce[i]);
            if (bounce_ev[i]) cudaEventDestroy(bounce_ev[i]);
            bounce[i] = nullptr;
            bounce_ev[i] = nullptr;
        }
        if (bits) cudaFree(bits);
        cudaFree(ctrl_mem);
        if (host_ctrl) cudaFreeHost(host_ctrl);
        host_ctrl = nullptr;
        if (keys) cudaFree(keys);
        if (parted) cudaFree(parted);
        if (bucket_scratch) cudaFree(bucket_scratch);
        if (wide) cudaFree(wide);
        if (width_scratch) cudaFree(width_scratch);
        if (small) cudaFree(small);
        small = nullptr;
        small_dirty = true;
        if (fused) cudaFree(fused);
        if (fused_saved) cudaFree(fused_saved);
        fused = nullptr;
        fused_dirty = true;
        fused_saved = nullptr;
        fused_saved_words = 0;
        wide = nullptr;
        wide_cap = 0;
        width_scratch = nullptr;
        parted = nullptr;
        parted_cap = 0;
        bucket_scratch = nullptr;
        if (stream) cudaStreamDestroy(stream);
        if (done) cudaEventDestroy(done);
        done = nullptr;
        bits = nullptr;
        ctrl_mem = nullptr;
        keys = nullptr;
        keys_cap = 0;
        stream = nullptr;
        ready = false;
    }
};

// ---- shared helpers (capi.cpp) ----
DeviceCtx& context_for(int device);
int visible_devices();
int current_device();
bool capturing(cudaStream_t stream);
void wait_done(DeviceCtx& ctx, cudaStream_t stream);
void record_done(DeviceCtx& ctx, cudaStream_t stream);
void preserve_pending(DeviceCtx& ctx, cudaStream_t stream);
bws_gpu::KernelTimer* active_timer();
cudaError_t launch_scan_any(const uint32_t* bits, uint64_t n_words, uint32_t key_base, uint32_t* out,
                            uint64_t cap, Ctrl* ctrl, unsigned long long* status,
                            unsigned long long* d_total, int clear, const bws_gpu::LaunchGeometry& geo,
                            cudaStream_t s);
void copy_parallel(void* dst, const void* src, size_t bytes);

// Brackets one launch with the kernel timer when it is enabled.
template <class F>
cudaError_t timed_launch(const char* name, cudaStream_t s, F&& launch) {
    bws_gpu::KernelTimer* t = active_timer();
    if (t) t->before(s);
    const cudaError_t err = launch();
    if (t) t->after(name, s);
    return err;
}

// ---- single-process multi-GPU sort (multi.cpp) ----
// Logical rank r runs on device multi_devices()[r] (a device may host
// several logical ranks: tests on one GPU). G = multi_devices().size().
int multi_rank_count();
std::vector<int> multi_devices();
// Sets the logical ranks (empty = single GPU); releases the previous ranks'
// buffers, streams and communicators. Throws config_error on a bad list.
void multi_set_devices(const std::vector<int>& devs);
// Sorts `count` distinct uint32 keys of a HOST array in place on the G
// configured devices (input-position shards, per-rank bitset, exchange,
// per-slice scan, each rank's slice written back at its offset). key_range
// 0 = derived. Returns false, leaving `data` untouched, if the keys repeat
// (the caller may fall back to the single-GPU multiset sort); throws
// data_error for keys >= key_range.
bool multi_sort_host(void* data, size_t count, uint64_t key_range);
void multi_release();

}  // namespace bws_host
