// Host side of libbitsort.so (B200 build): the reference's C ABI entry points
// (proj/src/capi.cpp) re-implemented over the sm_100a bitset kernels.
//
//   wrap()            <- proj/src/capi.cpp:19-41 (exception -> bws_status,
//                        thread-local message cleared on success)
//   bws_sort          <- proj/src/capi.cpp:186-197 -> dispatch.hpp:17-55
//                        (width 32, unsigned or signed (XOR bias), bitwise:
//                        every other combination is BWS_ERROR_CONFIG: there is
//                        no CPU fallback)
//   algorithm names   <- proj/src/capi.cpp:164-184, baselines.hpp:24-43
//
// Device state: one lazily created context per CUDA device (the calling
// thread's current device, or the device owning a device pointer) holding a
// cached 2^32-bit bitset that is all-zero between sorts (the direct path's K3
// clears every word it consumes), the control block + tile-status array, the
// bucket buffer and scratch of the bucketed path, a key staging buffer and
// pinned bounce buffers for host arrays, and an internal stream. Calls on one
// device are serialised by the context mutex; calls on different devices run
// concurrently. Multi-GPU: bws_sort on a host array runs on the devices set by
// bws_gpu_set_device_count / BITSORT_GPUS in this one process (multi.cpp);
// dist.py is the one-process-per-GPU alternative (torch.distributed).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <emmintrin.h>
#endif
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges are no-ops unless a tool attaches

#include "bitsort/bitsort.h"
#include "bitsort/bitsort_gpu.h"
#include "host_internal.h"
#include "kernels.h"

namespace bws_host {

thread_local std::string g_last_error;

template <class F>
bws_status wrap(F&& body) {
    try {
        body();
        g_last_error.clear();
        return BWS_OK;
    } catch (const config_error& e) {
        g_last_error = e.what();
        return BWS_ERROR_CONFIG;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        return BWS_ERROR_RANGE;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return BWS_ERROR_DATA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return BWS_ERROR_INTERNAL;
    } catch (...) {
        g_last_error = "unknown failure";
        return BWS_ERROR_INTERNAL;
    }
}

std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_scatter_mode{bws_gpu::kAuto};
std::atomic<int> g_path{-1};         // bws_path; -1 = not yet read from BITSORT_PATH

int current_path() {
    int p = g_path.load();
    if (p >= 0) return p;
    const char* env = std::getenv("BITSORT_PATH");
    p = BWS_PATH_AUTO;
    if (env && std::strcmp(env, "direct") == 0) p = BWS_PATH_DIRECT;
    if (env && std::strcmp(env, "bucketed") == 0) p = BWS_PATH_BUCKETED;
    if (env && std::strcmp(env, "fused") == 0) p = BWS_PATH_FUSED;
    if (env && std::strcmp(env, "fused_direct") == 0) p = BWS_PATH_FUSED_DIRECT;
    if (env && std::strcmp(env, "small") == 0) p = BWS_PATH_SMALL;
    g_path.store(p);
    return p;
}

// Persistent host thread pool for large memcpys (staging of pageable arrays
// through pinned bounce buffers). One copy at a time; the caller thread takes
// one slice itself.
class CopyPool {
   public:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        n_ = static_cast<int>(hw >= 16 ? 8 : (hw >= 4 ? hw / 2 : 1));
        if (const char* e = std::getenv("BITSORT_COPY_THREADS")) {  // staging copies of pageable arrays
            const int v = std::atoi(e);
            if (v >= 1 && v <= 64) n_ = v;
        }
        for (int i = 1; i < n_; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_start_.notify_all();
        for (auto& t : workers_) t.join();
    }
    void copy(void* dst, const void* src, size_t bytes) {
        if (bytes < (size_t(1) << 20) || n_ == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> one(copy_mu_);
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            pending_ = n_ - 1;
            ++gen_;
        }
        cv_start_.notify_all();
        part(0);
        std::unique_lock<std::mutex> lk(mu_);
        cv_done_.wait(lk, [this] { return pending_ == 0; });
    }

   private:
    // Streaming (non-temporal) stores for the staging copies: no
    // read-for-ownership of the destination lines (C2 through bws_sort on a
    // pageable array: 14.4-15.2 -> 13.4-13.8 ms). BITSORT_COPY_NT=0: memcpy.
    static void copy_piece(char* d, const char* s, size_t n) {
#if defined(__x86_64__)
        static const bool nt = [] {
            const char* e = std::getenv("BITSORT_COPY_NT");
            return !(e && e[0] == '0');
        }();
        if (nt && n >= 4096) {
            size_t head = (64 - (reinterpret_cast<uintptr_t>(d) & 63)) & 63;
            if (head) {
                std::memcpy(d, s, head);
                d += head;
                s += head;
                n -= head;
            }
            size_t i = 0;
            for (; i + 64 <= n; i += 64) {
                const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
                const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
                const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
                const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
                _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
                _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
                _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
                _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
            }
            _mm_sfence();
            if (i < n) std::memcpy(d + i, s + i, n - i);
            return;
        }
#endif
        std::memcpy(d, s, n);
    }
    void part(int i) {
        const size_t lo = (bytes_ * i / n_) & ~size_t(63), hi = i + 1 == n_ ? bytes_ : (bytes_ * (i + 1) / n_) & ~size_t(63);
        if (hi > lo) copy_piece(dst_ + lo, src_ + lo, hi - lo);
    }
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_start_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            lk.unlock();
            part(i);
            lk.lock();
            if (--pending_ == 0) cv_done_.notify_one();
        }
    }
    int n_ = 1;
    std::vector<std::thread> workers_;
    std::mutex mu_, copy_mu_;
    std::condition_variable cv_start_, cv_done_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
};

CopyPool& copy_pool() {
    static CopyPool pool;
    return pool;
}

void copy_parallel(void* dst, const void* src, size_t bytes) { copy_pool().copy(dst, src, bytes); }

// Per-kernel CUDA-event timing (bws_gpu_set_kernel_timing): events bracket
// each launch on its stream; bws_gpu_kernel_timings() resolves and sums them.
// Events are pooled per device (an event recorded on another device's stream
// fails), and the open "before" event is kept per stream, so timed sorts on
// different devices / threads never pair each other's events.
struct EventTimer final : bws_gpu::KernelTimer {
    std::mutex mu;
    std::atomic<bool> enabled{false};
    struct Rec {
        const char* name;
        int device;
        cudaEvent_t a, b;
    };
    std::vector<Rec> pending;
    std::map<int, std::vector<cudaEvent_t>> pool;     // per device
    std::map<cudaStream_t, std::pair<int, cudaEvent_t>> open;  // per stream: (device, event)

    static int device_now() {
        int d = 0;
        cuda_check(cudaGetDevice(&d), "cudaGetDevice(timer)");
        return d;
    }
    cudaEvent_t get(int device) {
        auto& p = pool[device];
        cudaEvent_t e = nullptr;
        if (!p.empty()) {
            e = p.back();
            p.pop_back();
        } else {
            cuda_check(cudaEventCreate(&e), "cudaEventCreate(timer)");
        }
        return e;
    }
    void before(cudaStream_t s) override {
        std::lock_guard<std::mutex> lock(mu);
        const int dev = device_now();
        cudaEvent_t e = get(dev);
        cuda_check(cudaEventRecord(e, s), "cudaEventRecord(timer)");
        auto it = open.find(s);
        if (it != open.end()) pool[it->second.first].push_back(it->second.second);  // unpaired: drop
        open[s] = {dev, e};
    }
    void after(const char* name, cudaStream_t s) override {
        std::lock_guard<std::mutex> lock(mu);
        auto it = open.find(s);
        if (it == open.end()) return;
        const int dev = it->second.first;
        cudaEvent_t b = get(dev);
        cuda_check(cudaEventRecord(b, s), "cudaEventRecord(timer)");
        pending.push_back({name, dev, it->second.second, b});
        open.erase(it);
    }
    std::string collect() {
        std::lock_guard<std::mutex> lock(mu);
        std::map<std::string, std::pair<uint64_t, double>> acc;
        for (const Rec& r : pending) {
            cuda_check(cudaEventSynchronize(r.b), "timer event");
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime");
            auto& slot = acc[r.name];
            slot.first += 1;
            slot.second += ms;
            pool[r.device].push_back(r.a);
            pool[r.device].push_back(r.b);
        }
        pending.clear();
        std::string out;
        for (const auto& [name, v] : acc)
            out += name + " " + std::to_string(v.first) + " " + std::to_string(v.second) + "\n";
        return out;
    }
};
EventTimer g_timer;

bws_gpu::KernelTimer* active_timer() { return g_timer.enabled.load() ? &g_timer : nullptr; }

// K3: v2 (TMA tiles, 128-wide lookback) unless the bitset is not 16-byte
// aligned or BITSORT_SCAN=v1 asks for the first version (A/B runs).
// Two-pass (tile counts first, then extraction without lookback) when the
// bitset is large relative to the output: the single-pass lookback chain
// stalls on sparse bitsets (measured C4 512 MiB: 584 us single pass).
// BITSORT_SCAN=v1|lookback|twopass forces a variant (A/B runs).
cudaError_t launch_scan_any(const uint32_t* bits, uint64_t n_words, uint32_t key_base, uint32_t* out,
                            uint64_t cap, Ctrl* ctrl, unsigned long long* status,
                            unsigned long long* d_total, int clear, const bws_gpu::LaunchGeometry& geo,
                            cudaStream_t s) {
    static const int mode = [] {
        const char* e = std::getenv("BITSORT_SCAN");
        if (!e) return 0;
        if (std::strcmp(e, "v1") == 0) return 1;
        if (std::strcmp(e, "lookback") == 0) return 2;
        if (std::strcmp(e, "twopass") == 0) return 3;
        return 0;
    }();
    int launches = 1;
    cudaError_t err;
    if (mode != 1 && bws_gpu::scan2_supported(bits)) {
        // two-pass only for large sparse bitsets (>= 16 MiB, at least 1 word per key);
        // small ones (C1) are latency-bound and one kernel is cheaper than three
        const bool two = n_words != 0 && (mode == 3 || (mode == 0 && n_words * 4 >= cap &&
                                                         n_words >= (uint64_t(1) << 22)));
        err = bws_gpu::launch_scan2(const_cast<uint32_t*>(bits), n_words, key_base, out, cap, ctrl,
                                    status, d_total, clear, geo, s, two ? 1 : 0, &launches);
    } else {
        err = bws_gpu::launch_scan(bits, n_words, key_base, out, cap, ctrl, status, d_total, clear, geo, s);
    }
    g_launches.fetch_add(static_cast<uint64_t>(launches - 1));  // callers count one
    return err;
}

constexpr int kMaxDevices = 64;
DeviceCtx g_ctx[kMaxDevices];

int visible_devices() {
    int count = 0;
    const cudaError_t err = cudaGetDeviceCount(&count);
    if (err != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw internal_error(
            std::string("no CUDA device available (") + cudaGetErrorString(err) +
            "); the B200 bitset sort has no CPU fallback");
    }
    return count;
}

DeviceCtx& context_for(int device) {
    if (device < 0 || device >= kMaxDevices) throw internal_error("device ordinal out of range");
    return g_ctx[device];
}

int current_device() {
    visible_devices();
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    return dev;
}

// Calls on one device share the context's buffers (control block, bucket
// buffer, cached bitset): each call's stream waits on `done`, recorded after
// the previous call's work. Under CUDA graph capture the graph's own
// dependencies order the captured work, and an event recorded outside the
// capture cannot be waited on inside it (nor a captured one outside), so both
// steps are skipped while `stream` is capturing.
bool capturing(cudaStream_t stream) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return st != cudaStreamCaptureStatusNone;
}
void wait_done(DeviceCtx& ctx, cudaStream_t stream) {
    if (!capturing(stream)) cuda_check(cudaStreamWaitEvent(stream, ctx.done, 0), "stream ordering");
}
void record_done(DeviceCtx& ctx, cudaStream_t stream) {
    if (!capturing(stream)) cuda_check(cudaEventRecord(ctx.done, stream), "cudaEventRecord");
}

// Every call that reuses the control block calls this once its stream waits on
// ctx.done: the pending async sort's control block is copied aside (stream-
// ordered, 64 bytes) so bws_gpu_sort_check still validates that sort. A new
// async sort supersedes the pending one instead (it clears `pending` first).
void preserve_pending(DeviceCtx& ctx, cudaStream_t stream) {
    if (!ctx.pending.active || ctx.pending.snapped) return;
    cuda_check(cudaMemcpyAsync(ctx.snap(), ctx.ctrl(), sizeof(Ctrl), cudaMemcpyDeviceToDevice, stream),
               "control block snapshot");
    ctx.pending.snapped = true;
}

// Queues one complete sort of `count` device-resident keys into `out` on
// `stream`: [bitset reset if dirty] -> control/status reset -> K2 -> K3.
// Caller holds ctx.mu. key_range == 0 derives the range from the keys (K2
// folds the max key; K3 scans (max >> 5) + 1 words).
void enqueue_direct(DeviceCtx& ctx, const uint32_t* keys, size_t count, uint32_t* out,
                    uint64_t key_range, cudaStream_t stream) {
    NvtxRange nvtx_range("bitsort:direct K2+K3");
    const bool derived = key_range == 0;
    const uint64_t words = derived ? 0 : (key_range + 31) / 32;
    wait_done(ctx, stream);
    preserve_pending(ctx, stream);
    ctx.ensure_bits();
    if (ctx.bits_dirty) {
        cuda_check(cudaMemsetAsync(ctx.bits, 0, kMaxWords * sizeof(uint32_t), stream),
                   "bitset reset");
        ctx.bits_dirty = false;
    }
    const size_t tiles = derived ? kMaxTiles : bws_gpu::scan_tiles(words);
    cuda_check(cudaMemsetAsync(ctx.ctrl_mem, 0, sizeof(Ctrl) + tiles * sizeof(unsigned long long),
                               stream),
               "control block reset");
    ctx.bits_dirty = true;
    cuda_check(timed_launch("bitset_scatter", stream,
                            [&] {
                                return bws_gpu::launch_scatter(
                                    keys, count, ctx.bits, derived ? kMaxKeyRange : key_range,
                                    ctx.ctrl(), g_scatter_mode.load(), ctx.geo, stream);
                            }),
               "bitset_scatter launch");
    g_launches.fetch_add(1);
    cuda_check(timed_launch("bitset_scan", stream,
                            [&] {
                                return launch_scan_any(ctx.bits, words, 0u, out, count, ctx.ctrl(),
                                                       ctx.status(), nullptr, /*clear=*/1, ctx.geo,
                                                       stream);
                            }),
               "bitset_scan launch");
    g_launches.fetch_add(1);
    ctx.bits_dirty = false;  // K3 zeroes every word it reads; all set bits lie in its range
    record_done(ctx, stream);
}

// Bucketed pipeline: [K0 max + host readback when no hint] -> KB1..KB4.
// Leaves the cached bitset untouched.
// key_lo: keys lie in [key_lo, key_lo + key_range) (range sorts). xr: keys
// are XORed with it on load and store (signed int32 sorts: 0x80000000).
// multiset: repeated keys are sorted too (packed layout + KB4m counting sort).
// K0 + host readback: the key range (max key + 1) of a sort without a hint,
// for the pipelines whose plan needs it on the host (bucketed, fused).
uint64_t derive_range(DeviceCtx& ctx, const uint32_t* keys, size_t count, cudaStream_t stream, uint32_t xr) {
    cuda_check(cudaMemsetAsync(ctx.ctrl_mem, 0, sizeof(Ctrl), stream), "control block reset");
    cuda_check(bws_gpu::launch_key_max(keys, count, ctx.ctrl(), ctx.geo, stream, xr), "key_max launch");
    g_launches.fetch_add(1);
    unsigned int mx = 0;
    cuda_check(cudaMemcpyAsync(&mx, &ctx.ctrl()->max_key, sizeof(mx), cudaMemcpyDeviceToHost, stream),
               "max key readback");
    cuda_check(cudaStreamSynchronize(stream), "key_max execution");
    return static_cast<uint64_t>(mx) + 1;
}

// Bucketed pipeline: [K0 max + host readback when no hint] -> KB1..KB4.
// Leaves the cached bitset untouched. Returns the key range it sorted with.
// key_lo: keys lie in [key_lo, key_lo + key_range) (range sorts). xr: keys
// are XORed with it on load and store (signed int32 sorts: 0x80000000).
// multiset: repeated keys are sorted too (packed layout + KB4m counting sort).
uint64_t enqueue_bucketed(DeviceCtx& ctx, const uint32_t* keys, size_t count, uint32_t* out,
                          uint64_t key_range, cudaStream_t stream, uint32_t key_lo = 0, uint32_t xr = 0,
                          bool multiset = false, int inplace_mode = 0) {
    NvtxRange nvtx_range("bitsort:bucketed KB1-KB4");
    wait_done(ctx, stream);
    preserve_pending(ctx, stream);
    if (key_range == 0) key_range = derive_range(ctx, keys, count, stream, xr);
    cuda_check(cudaMemsetAsync(ctx.ctrl_mem, 0, sizeof(Ctrl), stream), "control block reset");
    // signed sorts keep power-of-two bucket widths (the output XOR then
    // commutes with the in-bucket offsets)
    bws_gpu::BucketPlan plan =
        multiset ? bws_gpu::plan_multiset(key_range)
                 : bws_gpu::plan_buckets(key_range, xr ? 0 : ctx.geo.bucket_blocks[bws_gpu::MAX_BUCKET_SHIFT]);
    plan.map.lo = key_lo;
    plan.map.xr = xr;
    const size_t parted_cap = ctx.ensure_parted(count, plan);
    int launches = 0;
    cuda_check(bws_gpu::launch_bucket_sort(keys, count, key_range, out, ctx.parted, ctx.bucket_scratch,
                                           ctx.ctrl(), plan, ctx.geo, stream, &launches,
                                           active_timer(), nullptr, 0, parted_cap, multiset, nullptr, 0,
                                           inplace_mode),
               "bucketed sort launch");
    g_launches.fetch_add(static_cast<uint64_t>(launches));
    record_done(ctx, stream);
    return key_range;
}

// Whether a bucketed sort of `count` keys over key_range takes the slab
// layout (the only layout an in-place bws_sort can recover repeats from).
bool bucketed_slab(DeviceCtx& ctx, size_t count, uint64_t key_range, uint32_t xr) {
    const bws_gpu::BucketPlan plan =
        bws_gpu::plan_buckets(key_range, xr ? 0 : ctx.geo.bucket_blocks[bws_gpu::MAX_BUCKET_SHIFT]);
    const size_t cap = ctx.ensure_parted(count, plan);
    return bws_gpu::slab_in_use(plan, count, cap);
}

// KF: the single-launch fused sort (fused.cu) for key ranges whose bitset
// fits in the SMs' shared memory in <= 2 passes. key_lo as enqueue_bucketed.
bws_gpu::FusedPlan fused_plan(const DeviceCtx& ctx, uint64_t key_range, size_t count) {
    if (ctx.geo.fused_ctas <= 0 || count >= (size_t(1) << 32) || key_range == 0) return {};
    return bws_gpu::plan_fused(key_range, ctx.geo.fused_ctas, ctx.geo.fused_smem_limit);
}

// direct: the KD mode (keys ORed into the cached global bitset, a grid
// barrier, per-CTA slices counted and extracted); plan.P must be 1.
void enqueue_fused(DeviceCtx& ctx, const uint32_t* keys, size_t count, uint32_t* out, uint64_t key_range,
                   const bws_gpu::FusedPlan& plan, cudaStream_t stream, uint32_t key_lo = 0, bool direct = false) {
    NvtxRange nvtx_range(direct ? "bitsort:fused KD" : "bitsort:fused KF");
    wait_done(ctx, stream);
    preserve_pending(ctx, stream);
    ctx.ensure_fused(plan, stream);
    uint32_t* gbits = nullptr;
    if (direct) {
        ctx.ensure_bits();
        if (ctx.bits_dirty) {
            cuda_check(cudaMemsetAsync(ctx.bits, 0, kMaxWords * sizeof(uint32_t), stream), "bitset reset");
            ctx.bits_dirty = false;
        }
        gbits = ctx.bits;  // KD zeroes every word it takes: all-zero again afterwards
    }
    bws_gpu::KeySplit ks;
    const uintptr_t addr = reinterpret_cast<uintptr_t>(keys);
    size_t n_head = ((16 - (addr & 15)) & 15) / 4;
    if (n_head > count) n_head = count;
    ks.nv = (count - n_head) / 4;
    ks.body = reinterpret_cast<const uint4*>(keys + n_head);
    ks.head = keys;
    ks.n_head = static_cast<int>(n_head);
    ks.tail = keys + n_head + 4 * ks.nv;
    ks.n_tail = static_cast<int>(count - n_head - 4 * ks.nv);
    // BITSORT_KF_TRACE=1: per-CTA phase timestamps, summarised on stderr after
    // every fused sort (synchronous; a debugging aid, not for timing runs)
    static const bool trace_on = std::getenv("BITSORT_KF_TRACE") != nullptr;
    unsigned long long* trace = nullptr;
    if (trace_on) {
        static unsigned long long* buf = nullptr;
        if (!buf) cuda_check(cudaMalloc(&buf, bws_gpu::KF_MAXG * bws_gpu::KF_TRACE_WORDS * 8), "cudaMalloc(trace)");
        cuda_check(cudaMemsetAsync(buf, 0, bws_gpu::KF_MAXG * bws_gpu::KF_TRACE_WORDS * 8, stream), "trace reset");
        trace = buf;
    }
    cuda_check(timed_launch(direct ? "fused_direct" : "fused_sort", stream,
                            [&] {
                                return bws_gpu::launch_fused_sort(ks, key_range, key_lo, out, ctx.ctrl(),
                                                                  ctx.fused, ctx.fused_saved, plan, stream, trace,
                                                                  gbits);
                            }),
               "fused sort launch");
    g_launches.fetch_add(1);
    if (trace) {
        std::vector<unsigned long long> h(static_cast<size_t>(plan.G) * bws_gpu::KF_TRACE_WORDS);
        cuda_check(cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, stream), "trace readback");
        cuda_check(cudaStreamSynchronize(stream), "trace readback");
        const char* names[] = {"start", "prod0", "cons0", "prod1", "cons1", "counts", "end", "offs_in", "seen"};
        unsigned long long t0 = ~0ull;
        for (int c = 0; c < plan.G; ++c) t0 = std::min(t0, h[c * bws_gpu::KF_TRACE_WORDS]);
        std::fprintf(stderr, "[KF trace] n=%zu P=%d S=%u:", count, plan.P, plan.S);
        for (int ph = 0; ph < 9; ++ph) {
            std::vector<double> v;
            for (int c = 0; c < plan.G; ++c) {
                const unsigned long long t = h[c * bws_gpu::KF_TRACE_WORDS + ph];
                if (t) v.push_back((t - t0) / 1e3);
            }
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            std::fprintf(stderr, " %s %.1f/%.1f/%.1f", names[ph], v.front(), v[v.size() / 2], v.back());
        }
        std::fprintf(stderr, " us (min/med/max); producer clocks (median CTA, us at 1.9 GHz):");
        const char* pn[] = {"wait", "rank", "A", "scan", "scatter", "store"};
        for (int i = 0; i < 6; ++i) {
            std::vector<double> v;
            for (int c = 0; c < plan.G; ++c) v.push_back(h[c * bws_gpu::KF_TRACE_WORDS + 9 + i] / 1.9e3);
            std::sort(v.begin(), v.end());
            std::fprintf(stderr, " %s %.1f", pn[i], v[v.size() / 2]);
        }
        std::fprintf(stderr, "\n");
    }
    record_done(ctx, stream);
}

// KS: one cooperative launch for a small hinted sort (small.cu). The last CTA
// writes the control block, so nothing is reset before the launch.
// Returns false (nothing queued, KS disabled on this device from now on) when
// the driver refuses the cooperative launch — e.g. a context with fewer SMs
// than the device reports (MPS partitions): the caller takes the direct path.
bool enqueue_small(DeviceCtx& ctx, const uint32_t* keys, size_t count, uint32_t* out, uint64_t key_range,
                   const bws_gpu::SmallPlan& plan, cudaStream_t stream, uint32_t key_lo = 0) {
    NvtxRange nvtx_range("bitsort:small KS");
    wait_done(ctx, stream);
    preserve_pending(ctx, stream);
    ctx.ensure_bits();
    if (ctx.bits_dirty) {
        cuda_check(cudaMemsetAsync(ctx.bits, 0, kMaxWords * sizeof(uint32_t), stream), "bitset reset");
        ctx.bits_dirty = false;
    }
    ctx.ensure_small(stream);
    bws_gpu::KeySplit ks;
    const uintptr_t addr = reinterpret_cast<uintptr_t>(keys);
    size_t n_head = ((16 - (addr & 15)) & 15) / 4;
    if (n_head > count) n_head = count;
    ks.nv = (count - n_head) / 4;
    ks.body = reinterpret_cast<const uint4*>(keys + n_head);
    ks.head = keys;
    ks.n_head = static_cast<int>(n_head);
    ks.tail = keys + n_head + 4 * ks.nv;
    ks.n_tail = static_cast<int>(count - n_head - 4 * ks.nv);
    // BITSORT_KS_TRACE=1: per-CTA phase timestamps after every KS sort, on
    // stderr (synchronous; a debugging aid). BITSORT_KS_PREFETCH=0: no L2
    // prefetch of the bitset slices (A/B).
    static const bool trace_on = std::getenv("BITSORT_KS_TRACE") != nullptr;
    static const int prefetch = [] {
        const char* e = std::getenv("BITSORT_KS_PREFETCH");
        return e && e[0] == '0' ? 0 : 1;
    }();
    unsigned long long* trace = nullptr;
    const size_t trace_bytes = static_cast<size_t>(bws_gpu::KS_MAXG) * bws_gpu::KS_TRACE_WORDS * 8;
    if (trace_on) {
        static unsigned long long* buf = nullptr;
        if (!buf) cuda_check(cudaMalloc(&buf, trace_bytes), "cudaMalloc(trace)");
        cuda_check(cudaMemsetAsync(buf, 0, trace_bytes, stream), "trace reset");
        trace = buf;
    }
    const cudaError_t lerr = timed_launch("small_sort", stream, [&] {
        return bws_gpu::launch_small_sort(ks, key_range, key_lo, out, ctx.ctrl(), ctx.small, plan, ctx.bits, stream,
                                          trace, prefetch);
    });
    if (lerr == cudaErrorCooperativeLaunchTooLarge || lerr == cudaErrorNotSupported ||
        lerr == cudaErrorLaunchOutOfResources) {
        cudaGetLastError();
        ctx.geo.small_ctas = 0;
        return false;
    }
    cuda_check(lerr, "small sort launch");
    g_launches.fetch_add(1);
    if (trace) {
        std::vector<unsigned long long> h(static_cast<size_t>(plan.G) * bws_gpu::KS_TRACE_WORDS);
        cuda_check(cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, stream), "trace readback");
        cuda_check(cudaStreamSynchronize(stream), "trace readback");
        const char* names[] = {"start", "scattered", "barrier", "counted", "offsets", "end"};
        unsigned long long t0 = ~0ull;
        for (int c = 0; c < plan.G; ++c) t0 = std::min(t0, h[c * bws_gpu::KS_TRACE_WORDS]);
        std::fprintf(stderr, "[KS trace] n=%zu per=%u:", count, plan.per);
        for (int ph = 0; ph < 6; ++ph) {
            std::vector<double> v;
            for (int c = 0; c < plan.G; ++c) {
                const unsigned long long t = h[c * bws_gpu::KS_TRACE_WORDS + ph];
                if (t) v.push_back((t - t0) / 1e3);
            }
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            std::fprintf(stderr, " %s %.1f/%.1f/%.1f", names[ph], v.front(), v[v.size() / 2], v.back());
        }
        std::fprintf(stderr, " us (min/med/max over CTAs)\n");
    }
    record_done(ctx, stream);
    return true;
}

// One sort of distinct keys on the chosen pipeline. Returns the key range it
// sorted with (0: derived on the device by the direct pipeline, ctrl->max_key).
uint64_t enqueue_sort(DeviceCtx& ctx, const uint32_t* keys, size_t count, uint32_t* out,
                      uint64_t key_range, cudaStream_t stream, uint32_t key_lo = 0) {
    const int path = current_path();
    const bool coop = ctx.geo.fused_ctas > 0 && count < (size_t(1) << 32);
    // KD (fused direct) for hinted sorts of up to kFusedDirectMaxKeys keys
    // whose bitset slices fit in SMEM in one pass; the KF ring mode only
    // when asked for (BWS_PATH_FUSED: measured slower than BUCKETED on C2)
    if (coop && (path == BWS_PATH_FUSED_DIRECT ||
                 (path == BWS_PATH_AUTO && key_range != 0 && count >= kFusedMinKeys && count <= kFusedDirectMaxKeys))) {
        if (key_range == 0) {
            wait_done(ctx, stream);
            preserve_pending(ctx, stream);
            key_range = derive_range(ctx, keys, count, stream, 0);
        }
        const bws_gpu::FusedPlan plan = fused_plan(ctx, key_range, count);
        if (plan.ok && plan.P == 1) {
            enqueue_fused(ctx, keys, count, out, key_range, plan, stream, key_lo, /*direct=*/true);
            return key_range;
        }
    }
    if (coop && path == BWS_PATH_FUSED) {
        if (key_range == 0) {
            wait_done(ctx, stream);
            preserve_pending(ctx, stream);
            key_range = derive_range(ctx, keys, count, stream, 0);
        }
        const bws_gpu::FusedPlan plan = fused_plan(ctx, key_range, count);
        if (plan.ok) {
            enqueue_fused(ctx, keys, count, out, key_range, plan, stream, key_lo);
            return key_range;
        }
    }
    // KS for hinted sorts below the bucketed threshold whose range a CTA slice
    // holds in registers (C1: one launch instead of K2 + K3)
    if (ctx.geo.small_ctas > 0 && key_range != 0 &&
        (path == BWS_PATH_SMALL ||
         ((path == BWS_PATH_AUTO || path == BWS_PATH_FUSED || path == BWS_PATH_FUSED_DIRECT) &&
          count < kBucketedMinKeys && key_range <= kSmallMaxRange))) {
        const bws_gpu::SmallPlan plan = bws_gpu::plan_small(key_range, ctx.geo.small_ctas);
        if (plan.ok && count < (size_t(1) << 32) &&
            enqueue_small(ctx, keys, count, out, key_range, plan, stream, key_lo))
            return key_range;
    }
    // FUSED / FUSED_DIRECT / SMALL with a range they cannot hold fall back to AUTO's choice
    const bool bucketed = key_lo != 0 || (count < (size_t(1) << 32) &&
                                          (path == BWS_PATH_BUCKETED ||
                                           (path != BWS_PATH_DIRECT && count >= kBucketedMinKeys)));
    if (bucketed) return enqueue_bucketed(ctx, keys, count, out, key_range, stream, key_lo);
    enqueue_direct(ctx, keys, count, out, key_range, stream);
    return key_range;
}

// Synchronises and reads the control block back.
Ctrl read_ctrl(DeviceCtx& ctx, cudaStream_t stream) {
    // one stream-ordered copy into pinned memory and one wait (a blocking
    // cudaMemcpy after the synchronise cost a second host round trip)
    cuda_check(cudaMemcpyAsync(ctx.host_ctrl, ctx.ctrl(), sizeof(Ctrl), cudaMemcpyDeviceToHost, stream),
               "control block readback");
    cuda_check(cudaStreamSynchronize(stream), "sort execution");
    const Ctrl c = *ctx.host_ctrl;
    if (c.error != 0) {  // KF ring / chunk-table protocol timeout: reset the ring state
        ctx.fused_dirty = true;
        ctx.small_dirty = true;
        ctx.bits_dirty = true;  // a KD / KS sort may have stopped before taking its slices
        throw internal_error("sort protocol timeout (a kernel gave up waiting; state reset)");
    }
    return c;
}

void throw_bad_keys(const Ctrl& c, uint64_t key_range) {
    if (c.bad_keys != 0)
        throw data_error(std::to_string(c.bad_keys) + " key(s) not below the key range " +
                         std::to_string(key_range));
}

// Synchronises and turns the control block into a status: out-of-range keys
// or duplicates (fewer set bits than keys) are BWS_ERROR_DATA.
uint64_t validate(DeviceCtx& ctx, size_t count, uint64_t key_range, cudaStream_t stream) {
    const Ctrl c = read_ctrl(ctx, stream);
    throw_bad_keys(c, key_range);
    if (c.total != count)
        throw data_error("keys are not distinct: " + std::to_string(count) + " keys, " +
                         std::to_string(c.total) +
                         " distinct (the bitset sort requires distinct keys)");
    return c.total;
}

void check_range(uint64_t key_range) {
    if (key_range > kMaxKeyRange)
        throw std::out_of_range("key range " + std::to_string(key_range) +
                                " exceeds 2^32 for 32-bit keys");
}

// Pageable host array -> device: 16 MiB chunks through two pinned bounce
// buffers; the multi-threaded host copy of chunk i+1 overlaps the DMA of
// chunk i (the driver's own pageable path measured 4x slower than pinned).
void stage_to_device(DeviceCtx& ctx, void* dev, const void* host, size_t bytes) {
    NvtxRange nvtx_range("bitsort:host-to-device");
    ctx.ensure_bounce();
    for (size_t off = 0, i = 0; off < bytes; off += kStageChunk, ++i) {
        const int b = static_cast<int>(i & 1);
        const size_t len = bytes - off < kStageChunk ? bytes - off : kStageChunk;
        cuda_check(cudaEventSynchronize(ctx.bounce_ev[b]), "staging buffer reuse");
        copy_pool().copy(ctx.bounce[b], static_cast<const char*>(host) + off, len);
        cuda_check(cudaMemcpyAsync(static_cast<char*>(dev) + off, ctx.bounce[b], len,
                                   cudaMemcpyHostToDevice, ctx.stream),
                   "host-to-device copy");
        cuda_check(cudaEventRecord(ctx.bounce_ev[b], ctx.stream), "cudaEventRecord");
    }
}

// Device -> pageable host array, the mirror image (DMA of chunk i+1 overlaps
// the host copy of chunk i).
void stage_to_host(DeviceCtx& ctx, void* host, const void* dev, size_t bytes) {
    NvtxRange nvtx_range("bitsort:device-to-host");
    ctx.ensure_bounce();
    const size_t nch = (bytes + kStageChunk - 1) / kStageChunk;
    auto issue = [&](size_t i) {
        const int b = static_cast<int>(i & 1);
        const size_t off = i * kStageChunk;
        const size_t len = bytes - off < kStageChunk ? bytes - off : kStageChunk;
        cuda_check(cudaMemcpyAsync(ctx.bounce[b], static_cast<const char*>(dev) + off, len,
                                   cudaMemcpyDeviceToHost, ctx.stream),
                   "device-to-host copy");
        cuda_check(cudaEventRecord(ctx.bounce_ev[b], ctx.stream), "cudaEventRecord");
    };
    for (size_t i = 0; i < nch && i < 2; ++i) issue(i);
    for (size_t i = 0; i < nch; ++i) {
        const int b = static_cast<int>(i & 1);
        const size_t off = i * kStageChunk;
        const size_t len = bytes - off < kStageChunk ? bytes - off : kStageChunk;
        cuda_check(cudaEventSynchronize(ctx.bounce_ev[b]), "device-to-host copy");
        copy_pool().copy(static_cast<char*>(host) + off, ctx.bounce[b], len);
        if (i + 2 < nch) issue(i + 2);
    }
}

// The drop-in sort on the calling thread's current device (or the device
// owning `data` when it is device memory). Host arrays are staged through the
// context's device buffer; they are written back only after validation, so a
// rejected input is left untouched.
// multiset (bws_sort): an input with repeated keys is sorted too, like the
// reference's bws_sort sorts any input. The bitset pass detects the repeats
// (fewer set bits than keys) and the sort is redone from the untouched input
// by the counting-sort pipeline (KB1-KB3 packed + KB4m). Device arrays are
// then sorted out of place into the context's key buffer and copied back, so
// the original survives the detection. Without multiset (the key-range
// extension) repeated keys are BWS_ERROR_DATA.
// Host arrays below this many keys stay on one GPU even when G > 1 devices
// are configured (env BITSORT_MULTI_MIN_KEYS; tests lower it).
size_t multi_min_keys() {
    const char* e = std::getenv("BITSORT_MULTI_MIN_KEYS");
    return e ? static_cast<size_t>(std::strtoull(e, nullptr, 10)) : (size_t(1) << 20);
}

// The reference's counting_sort (baselines.hpp:95-110) rejects a key span
// max - min >= 2^26 with std::out_of_range (BWS_ERROR_RANGE) before sorting.
[[noreturn]] void throw_span(uint64_t diff, uint64_t limit) {
    throw std::out_of_range("counting_sort: key span " + std::to_string(diff) + "+1 exceeds the limit of " +
                            std::to_string(limit) + " keys");
}

// BITSORT_SPECULATE=0: every in-place device-array sort without a hint runs K0.
bool speculate_range() {
    static const bool on = [] {
        const char* e = std::getenv("BITSORT_SPECULATE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// The range planned for after a sort whose keys had `range`: rounded up to 1/64
// of the enclosing power of two, so the next array of the same kind (its
// largest key a little above or below) still fits, capped at 2^32.
uint64_t spec_round(uint64_t range) {
    if (range == 0) return 0;
    uint64_t p = 1;
    while (p < range) p <<= 1;
    const uint64_t g = p >> 6 ? p >> 6 : 1;
    const uint64_t r = (range + g - 1) / g * g;
    return r > kMaxKeyRange ? kMaxKeyRange : r;
}

// span_limit != 0 (BWS_ALG_COUNTING): K0 first folds min and max on the
// device; a span >= span_limit is BWS_ERROR_RANGE with the data untouched,
// otherwise max + 1 becomes the sort's key-range hint.
void sort_u32(void* data, size_t count, uint64_t key_range, uint32_t xr = 0, bool multiset = false,
              uint64_t span_limit = 0) {
    NvtxRange nvtx_range("bitsort:bws_sort u32");
    check_range(key_range);
    if (count == 0) return;
    visible_devices();
    cudaPointerAttributes attr{};
    cudaError_t perr = cudaPointerGetAttributes(&attr, data);
    if (perr != cudaSuccess) {
        cudaGetLastError();
        attr.type = cudaMemoryTypeUnregistered;
    }
    const bool on_device = attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
    int device = 0;
    if (on_device) {
        device = attr.device;
    } else {
        cuda_check(cudaGetDevice(&device), "cudaGetDevice");
    }
    // a host array of unsigned keys on G > 1 configured devices: the
    // single-process multi-GPU sort (multi.cpp, which locks every device
    // context itself, so this runs before ctx.mu is taken); repeated keys come
    // back untouched and take the single-GPU counting pass below
    if (!on_device && xr == 0 && span_limit == 0 && count >= multi_min_keys() && multi_rank_count() > 1) {
        if (multi_sort_host(data, count, key_range)) return;
        if (!multiset)
            throw data_error("keys are not distinct: " + std::to_string(count) +
                             " keys (the bitset sort requires distinct keys)");
    }
    DeviceCtx& ctx = context_for(device);
    std::lock_guard<std::mutex> lock(ctx.mu);
    int prev = 0;
    cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    struct restore_device {
        int d;
        ~restore_device() { cudaSetDevice(d); }
    } restore{prev};
    ctx.init(device);
    uint32_t* keys = static_cast<uint32_t*>(data);
    const uint64_t hinted_range = key_range;  // 0: the caller gave no range
    auto check_span = [&](const uint32_t* dk) {
        if (span_limit == 0) return;
        wait_done(ctx, ctx.stream);
        preserve_pending(ctx, ctx.stream);
        cuda_check(cudaMemsetAsync(ctx.ctrl_mem, 0, sizeof(Ctrl), ctx.stream), "control block reset");
        cuda_check(bws_gpu::launch_key_max(dk, count, ctx.ctrl(), ctx.geo, ctx.stream, xr), "key_max launch");
        g_launches.fetch_add(1);
        const Ctrl c = read_ctrl(ctx, ctx.stream);
        record_done(ctx, ctx.stream);
        const uint64_t mn = static_cast<uint32_t>(~c.min_inv), mx = c.max_key;
        if (mx - mn >= span_limit) throw_span(mx - mn, span_limit);
        key_range = mx + 1;
    };
    // signed keys (xr) always take the bucketed pipeline, which applies the XOR
    uint64_t sorted_range = key_range;  // the range the bitset pass used (0: derived on the device)
    // Small unhinted sorts (count < 2^21, AUTO): K2 + K3 derive the range on the
    // device; once a sort has told the host its keys' range (K2 and KS fold the
    // largest key), the next one runs KS planned for that range — one launch
    // instead of two. Keys beyond it are counted as bad: the pass is redone
    // with K2 + K3 (the device copy is intact or re-uploaded).
    bool small_spec = false;  // the bitset pass ran KS on the speculated range
    const bool small_unhinted = hinted_range == 0 && xr == 0 && span_limit == 0 && count < kBucketedMinKeys &&
                                current_path() == BWS_PATH_AUTO;
    auto enqueue = [&](const uint32_t* in, uint32_t* out) {
        small_spec = false;
        if (small_unhinted && key_range == 0 && ctx.geo.small_ctas > 0 && speculate_range() &&
            ctx.spec_small != 0 && ctx.spec_small <= kSmallMaxRange) {
            const bws_gpu::SmallPlan plan = bws_gpu::plan_small(ctx.spec_small, ctx.geo.small_ctas);
            if (plan.ok && enqueue_small(ctx, in, count, out, ctx.spec_small, plan, ctx.stream)) {
                sorted_range = ctx.spec_small;
                small_spec = true;
                return;
            }
        }
        if (xr) {
            if (count >= (size_t(1) << 32)) throw std::out_of_range("signed sorts take fewer than 2^32 keys");
            sorted_range = enqueue_bucketed(ctx, in, count, out, key_range, ctx.stream, 0, xr);
        } else {
            sorted_range = enqueue_sort(ctx, in, count, out, key_range, ctx.stream);
        }
    };
    // after the bitset pass: true if the keys repeat and the counting-sort
    // pass must run (its key range: the max key the first pass folded)
    uint64_t ms_range = 0;
    // restore_input: brings `in` back when the pass sorted in place (host
    // arrays: upload again); called before a pass is redone
    auto needs_multiset = [&](const uint32_t* in, uint32_t* out, const std::function<void()>& restore_input) {
        Ctrl c = read_ctrl(ctx, ctx.stream);
        if (small_spec && c.bad_keys != 0) {  // the keys outgrew the speculated range
            ctx.spec_small = 0;
            restore_input();
            enqueue(in, out);
            c = read_ctrl(ctx, ctx.stream);
        }
        throw_bad_keys(c, key_range ? key_range : kMaxKeyRange);
        if (small_unhinted && key_range == 0) {
            const uint64_t r = spec_round(static_cast<uint64_t>(c.max_key) + 1);
            ctx.spec_small = r <= kSmallMaxRange ? r : 0;
        }
        if (c.total == count) return false;
        if (!multiset)
            throw data_error("keys are not distinct: " + std::to_string(count) + " keys, " +
                             std::to_string(c.total) + " distinct (the bitset sort requires distinct keys)");
        if (count >= (size_t(1) << 32))
            throw std::out_of_range("sorting repeated keys takes fewer than 2^32 keys");
        ms_range = key_range ? key_range : sorted_range ? sorted_range : static_cast<uint64_t>(c.max_key) + 1;
        return true;
    };
    auto enqueue_multiset = [&](const uint32_t* in, uint32_t* out) {
        enqueue_bucketed(ctx, in, count, out, ms_range, ctx.stream, 0, xr, /*multiset=*/true);
        validate(ctx, count, ms_range, ctx.stream);
    };
    if (on_device) {
        check_span(keys);
        if (!multiset) {
            enqueue(keys, keys);
            validate(ctx, count, key_range, ctx.stream);
            return;
        }
        // In place when the bucketed slab pipeline takes the keys: KB3 reads
        // every key before KB4 writes any output, a slab that lost runs makes
        // KB4 write nothing (the keys stay intact for the counting pass), and
        // otherwise the slabs hold the exact key multiset, from which KB4m
        // redoes a sort whose keys repeat. Other pipelines sort out of place.
        const int path = current_path();
        if (count >= kBucketedMinKeys && count < (size_t(1) << 32) &&
            (path == BWS_PATH_AUTO || path == BWS_PATH_BUCKETED)) {
            wait_done(ctx, ctx.stream);
            preserve_pending(ctx, ctx.stream);
            // No hint: instead of K0 (a read of every key plus a host round
            // trip before KB3 can be planned) the sort is planned for the range
            // the previous such sort's keys had (KB3 folds the largest key it
            // sees, ctrl->max_key). Keys beyond a speculated range are counted
            // as bad and make the in-place KB4 write nothing, so a miss costs
            // one KB3 and is redone from the intact keys with K0's range.
            bool speculated = false;
            if (key_range == 0) {
                // (two misses in a row — a caller alternating between ranges —
                // switch speculation off for the next 16 sorts: a miss costs a KB3)
                if (ctx.spec_cooldown > 0) --ctx.spec_cooldown;
                if (ctx.spec_range != 0 && ctx.spec_cooldown == 0 && speculate_range()) {
                    key_range = ctx.spec_range;
                    speculated = true;
                } else {
                    key_range = derive_range(ctx, keys, count, ctx.stream, xr);
                }
            }
            if (speculated && !bucketed_slab(ctx, count, key_range, xr)) {
                key_range = derive_range(ctx, keys, count, ctx.stream, xr);
                speculated = false;
            }
            if (bucketed_slab(ctx, count, key_range, xr)) {
                enqueue_bucketed(ctx, keys, count, keys, key_range, ctx.stream, 0, xr, false, /*inplace=*/1);
                Ctrl c = read_ctrl(ctx, ctx.stream);
                if (speculated && c.bad_keys == 0) ctx.spec_misses = 0;
                if (speculated && c.bad_keys != 0) {  // the keys outgrew the speculated range
                    if (++ctx.spec_misses >= 2) {
                        ctx.spec_misses = 0;
                        ctx.spec_cooldown = 16;
                    }
                    ctx.spec_range = 0;
                    key_range = derive_range(ctx, keys, count, ctx.stream, xr);
                    speculated = false;
                    if (!bucketed_slab(ctx, count, key_range, xr)) {
                        ctx.spec_range = spec_round(key_range);
                        goto out_of_place;
                    }
                    enqueue_bucketed(ctx, keys, count, keys, key_range, ctx.stream, 0, xr, false, /*inplace=*/1);
                    c = read_ctrl(ctx, ctx.stream);
                }
                throw_bad_keys(c, key_range);
                if (hinted_range == 0) ctx.spec_range = spec_round(static_cast<uint64_t>(c.max_key) + 1);
                if (c.total == count) return;
                if (count >= (size_t(1) << 32)) throw std::out_of_range("sorting repeated keys takes fewer than 2^32 keys");
                ms_range = key_range;
                if (c.overflow) {  // nothing written: the counting pass from the keys
                    enqueue_multiset(keys, keys);
                    return;
                }
                enqueue_bucketed(ctx, keys, count, keys, key_range, ctx.stream, 0, xr, false, /*recover=*/2);
                validate(ctx, count, key_range, ctx.stream);
                return;
            }
        }
    out_of_place:
        ctx.ensure_keys(count);
        enqueue(keys, ctx.keys);
        if (needs_multiset(keys, ctx.keys, [] {})) {
            enqueue_multiset(keys, keys);
            return;
        }
        cuda_check(cudaMemcpyAsync(keys, ctx.keys, count * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx.stream),
                   "device-to-device copy");
        cuda_check(cudaStreamSynchronize(ctx.stream), "device-to-device copy");
        return;
    }
    ctx.ensure_keys(count);
    const size_t bytes = count * sizeof(uint32_t);
    const bool pinned = attr.type == cudaMemoryTypeHost;
    auto upload = [&] {
        if (pinned) {
            cuda_check(cudaMemcpyAsync(ctx.keys, data, bytes, cudaMemcpyHostToDevice, ctx.stream),
                       "host-to-device copy");
        } else {
            stage_to_device(ctx, ctx.keys, data, bytes);
        }
    };
    upload();
    check_span(ctx.keys);
    enqueue(ctx.keys, ctx.keys);
    if (needs_multiset(ctx.keys, ctx.keys, upload)) {
        upload();  // the host array is untouched until the write-back
        enqueue_multiset(ctx.keys, ctx.keys);
    }
    if (pinned) {
        cuda_check(cudaMemcpyAsync(data, ctx.keys, bytes, cudaMemcpyDeviceToHost, ctx.stream),
                   "device-to-host copy");
        cuda_check(cudaStreamSynchronize(ctx.stream), "device-to-host copy");
    } else {
        stage_to_host(ctx, data, ctx.keys, bytes);
    }
}

// 8-, 16- and 64-bit keys (the reference's with_width arms, dispatch.hpp:17-40),
// on the GPU: 8/16-bit keys by a counting sort over the type's range
// (widths.cu KW1-KW3, repeats included); 64-bit keys whose biased span
// max - min is below 2^32 narrowed to u32 offsets, sorted by the 32-bit
// pipeline (repeats redone by the counting pass) and widened back. Wider
// 64-bit spans are BWS_ERROR_CONFIG (no CPU fallback).
void sort_other_width(void* data, size_t count, uint32_t width, int is_unsigned, uint64_t span_limit = 0) {
    NvtxRange nvtx_range("bitsort:bws_sort other width");
    if (count == 0) return;
    visible_devices();
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, data) != cudaSuccess) {
        cudaGetLastError();
        attr.type = cudaMemoryTypeUnregistered;
    }
    const bool on_device = attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
    int device = 0;
    if (on_device)
        device = attr.device;
    else
        cuda_check(cudaGetDevice(&device), "cudaGetDevice");
    DeviceCtx& ctx = context_for(device);
    std::lock_guard<std::mutex> lock(ctx.mu);
    int prev = 0;
    cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    struct restore_device {
        int d;
        ~restore_device() { cudaSetDevice(d); }
    } restore{prev};
    ctx.init(device);
    const size_t bytes = count * (width / 8);
    // host arrays: keys at wide[0, bytes); every 64-bit sort also gets a
    // second array of `bytes` (the radix sort's ping-pong partner)
    const size_t partner = width == 64 ? bytes : 0;
    void* scratch_owner = ctx.ensure_wide((on_device ? 0 : bytes) + partner + 16);
    void* dev = on_device ? data : scratch_owner;
    void* other = static_cast<unsigned char*>(scratch_owner) + (on_device ? 0 : bytes);
    const bool pinned = attr.type == cudaMemoryTypeHost;
    cudaStream_t s = ctx.stream;
    wait_done(ctx, s);
    auto upload = [&] {
        if (on_device) return;
        if (pinned)
            cuda_check(cudaMemcpyAsync(dev, data, bytes, cudaMemcpyHostToDevice, s), "host-to-device copy");
        else
            stage_to_device(ctx, dev, data, bytes);
    };
    upload();
    if (width == 8 || width == 16) {
        int launches = 0;
        cuda_check(bws_gpu::launch_sort_small(dev, count, static_cast<int>(width), is_unsigned, ctx.width_scratch,
                                              ctx.geo, s, &launches, active_timer()),
                   "counting sort launch");
        g_launches.fetch_add(static_cast<uint64_t>(launches));
    } else {
        const uint64_t* k64 = static_cast<const uint64_t*>(dev);
        cuda_check(bws_gpu::launch_minmax64(k64, count, is_unsigned, ctx.width_scratch, ctx.geo, s), "min/max launch");
        g_launches.fetch_add(1);
        uint64_t mm[2] = {0, 0};
        cuda_check(cudaMemcpyAsync(mm, ctx.width_scratch, sizeof mm, cudaMemcpyDeviceToHost, s), "min/max readback");
        cuda_check(cudaStreamSynchronize(s), "min/max");
        if (span_limit && mm[1] - mm[0] >= span_limit) throw_span(mm[1] - mm[0], span_limit);
        if (mm[1] - mm[0] >= (uint64_t(1) << 32)) {
            // a span beyond the bitset sort's 2^32: stable LSD radix passes over
            // the 8-bit digits on which the keys differ
            if (count >= (size_t(1) << 32)) throw std::out_of_range("64-bit radix sorts take fewer than 2^32 keys");
            if (bws_gpu::radix64_scratch_bytes(ctx.geo) > bws_gpu::width_scratch_bytes())
                throw std::runtime_error("radix scratch too small");
            cuda_check(bws_gpu::launch_radix64_hist(k64, count, is_unsigned, ctx.width_scratch, ctx.geo, s),
                       "radix histogram launch");
            g_launches.fetch_add(1);
            std::vector<uint64_t> hist(8 * 256);
            cuda_check(cudaMemcpyAsync(hist.data(), ctx.width_scratch, hist.size() * sizeof(uint64_t),
                                       cudaMemcpyDeviceToHost, s),
                       "radix histogram readback");
            cuda_check(cudaStreamSynchronize(s), "radix histogram");
            std::vector<int> digits;
            for (int d = 0; d < 8; ++d)
                if (*std::max_element(hist.begin() + 256 * d, hist.begin() + 256 * (d + 1)) != count)
                    digits.push_back(d);
            const uint64_t bias = is_unsigned ? 0 : (uint64_t(1) << 63);
            uint64_t* cur = static_cast<uint64_t*>(dev);
            uint64_t* nxt = static_cast<uint64_t*>(other);
            for (size_t j = 0; j < digits.size(); ++j) {
                cuda_check(bws_gpu::launch_radix64_pass(cur, nxt, count, digits[j], j == 0 ? bias : 0,
                                                        j + 1 == digits.size() ? bias : 0, ctx.width_scratch,
                                                        ctx.geo, s),
                           "radix pass launch");
                g_launches.fetch_add(3);
                std::swap(cur, nxt);
            }
            if (cur != dev)
                cuda_check(cudaMemcpyAsync(dev, cur, bytes, cudaMemcpyDeviceToDevice, s), "radix result copy");
        } else {
            const uint64_t range = mm[1] - mm[0] + 1;
            ctx.ensure_keys(count);
            auto narrow = [&] {
                cuda_check(bws_gpu::launch_narrow64(k64, count, is_unsigned, ctx.width_scratch, ctx.keys, ctx.geo, s),
                           "narrowing launch");
                g_launches.fetch_add(1);
            };
            narrow();
            enqueue_sort(ctx, ctx.keys, count, ctx.keys, range, s);
            const Ctrl c = read_ctrl(ctx, s);
            if (c.total != count) {  // repeated keys: the counting pass, from the untouched 64-bit keys
                if (count >= (size_t(1) << 32))
                    throw std::out_of_range("sorting repeated keys takes fewer than 2^32 keys");
                narrow();
                enqueue_bucketed(ctx, ctx.keys, count, ctx.keys, range, s, 0, 0, /*multiset=*/true);
                validate(ctx, count, range, s);
            }
            cuda_check(bws_gpu::launch_widen64(ctx.keys, count, is_unsigned, ctx.width_scratch,
                                               static_cast<uint64_t*>(dev), ctx.geo, s),
                       "widening launch");
            g_launches.fetch_add(1);
        }
    }
    if (on_device) {
        cuda_check(cudaStreamSynchronize(s), "sort execution");
    } else if (pinned) {
        cuda_check(cudaMemcpyAsync(data, dev, bytes, cudaMemcpyDeviceToHost, s), "device-to-host copy");
        cuda_check(cudaStreamSynchronize(s), "device-to-host copy");
    } else {
        cuda_check(cudaStreamSynchronize(s), "sort execution");
        stage_to_host(ctx, data, dev, bytes);
    }
    record_done(ctx, s);
}

const char* algorithm_name_of(bws_algorithm a) {
    switch (a) {
        case BWS_ALG_BITWISE: return "bitwise";
        case BWS_ALG_BITWISE_SKIP_EMPTY: return "bitwise_skip_empty";
        case BWS_ALG_INSERTION: return "insertion";
        case BWS_ALG_MERGE: return "merge";
        case BWS_ALG_COUNTING: return "counting";
        case BWS_ALG_PLATFORM: return "platform";
    }
    return "unknown";
}

}  // namespace bws_host

using namespace bws_host;

extern "C" {

const char* bws_version(void) { return "1.0.0"; }

const char* bws_last_error(void) { return g_last_error.c_str(); }

const char* bws_algorithm_name(bws_algorithm algorithm) { return algorithm_name_of(algorithm); }

bws_status bws_algorithm_from_name(const char* name, bws_algorithm* out) {
    return wrap([&] {
        if (name == nullptr) throw config_error("null algorithm name");
        if (out == nullptr) throw config_error("null output pointer");
        for (int id = BWS_ALG_BITWISE; id <= BWS_ALG_PLATFORM; ++id) {
            const auto a = static_cast<bws_algorithm>(id);
            if (std::strcmp(name, algorithm_name_of(a)) == 0) {
                *out = a;
                return;
            }
        }
        throw config_error("unknown algorithm '" + std::string(name) + "'");
    });
}

bws_status bws_sort(void* data, size_t count, uint32_t width, int is_unsigned,
                    bws_algorithm algorithm) {
    return wrap([&] {
        if (count > 0 && data == nullptr) throw data_error("null data with nonzero count");
        if (static_cast<int>(algorithm) < BWS_ALG_BITWISE ||
            static_cast<int>(algorithm) > BWS_ALG_PLATFORM)
            throw config_error("unknown algorithm id");
        if (width != 8 && width != 16 && width != 32 && width != 64)
            throw config_error("unsupported width " + std::to_string(width) +
                               " (expected 8, 16, 32, or 64)");
        // Nothing to sort: the reference returns OK for any valid (width,
        // signedness, algorithm) here (test_capi.cpp:95), so do we.
        if (count == 0) return;
        // bitsort.h:86-88: the array holds naturally aligned keys of `width` bits
        if (reinterpret_cast<uintptr_t>(data) % (width / 8) != 0)
            throw data_error("data is not aligned to its " + std::to_string(width) + "-bit keys");
        // Every algorithm id yields the same bytes (a sort's output is unique),
        // so all of them run on the GPU pipelines (run_algorithm,
        // dispatch.hpp:42-55). COUNTING keeps the reference's one behavioural
        // difference: a key span >= 2^26 is BWS_ERROR_RANGE
        // (counting_sort_max_range_default, baselines.hpp:95-110).
        const uint64_t span_limit = algorithm == BWS_ALG_COUNTING ? (uint64_t(1) << 26) : 0;
        if (width != 32) {
            sort_other_width(data, count, width, is_unsigned, span_limit);
            return;
        }
        // signed int32: x ^ 0x80000000 maps the signed order onto the unsigned
        // one (the reference splits negatives and non-negatives instead,
        // bitsort.hpp:131-152); the same XOR maps the sorted keys back
        sort_u32(data, count, 0, is_unsigned ? 0u : 0x80000000u, /*multiset=*/true, span_limit);
    });
}

bws_status bws_sort_u32_range(void* data, size_t count, uint64_t key_range) {
    return wrap([&] {
        if (count > 0 && data == nullptr) throw data_error("null data with nonzero count");
        if (key_range == 0 && count > 0) throw std::out_of_range("key range 0 holds no keys");
        sort_u32(data, count, key_range);
    });
}

bws_status bws_gpu_sort_device_async(const uint32_t* keys, size_t count, uint32_t* out,
                                     uint64_t key_range, void* stream) {
    return wrap([&] {
        if (count > 0 && (keys == nullptr || out == nullptr))
            throw data_error("null device pointer with nonzero count");
        check_range(key_range);
        const int dev = current_device();
        DeviceCtx& ctx = context_for(dev);
        std::lock_guard<std::mutex> lock(ctx.mu);
        ctx.init(dev);
        ctx.pending.active = false;  // superseded by this sort
        if (count == 0) return;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        // no hint: the direct pipeline derives the range on the device (K2
        // folds the max key, K3 scans up to it) with no host round trip, so
        // the call stays stream-ordered and capturable; the bucketed
        // pipeline's plan needs the range on the host
        if (key_range == 0)
            enqueue_direct(ctx, keys, count, out, 0, s);
        else
            enqueue_sort(ctx, keys, count, out, key_range, s);
        ctx.pending = {true, s, count, key_range, false};
    });
}

bws_status bws_gpu_sort_range_device_async(const uint32_t* keys, size_t count, uint32_t* out,
                                           uint32_t key_lo, uint64_t key_range, void* stream) {
    return wrap([&] {
        if (count > 0 && (keys == nullptr || out == nullptr))
            throw data_error("null device pointer with nonzero count");
        if (key_range == 0 || static_cast<uint64_t>(key_lo) + key_range > kMaxKeyRange)
            throw std::out_of_range("key range [" + std::to_string(key_lo) + ", " +
                                    std::to_string(static_cast<uint64_t>(key_lo) + key_range) +
                                    ") is empty or exceeds 2^32");
        const int dev = current_device();
        DeviceCtx& ctx = context_for(dev);
        std::lock_guard<std::mutex> lock(ctx.mu);
        ctx.init(dev);
        ctx.pending.active = false;  // superseded by this sort
        if (count == 0) return;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (key_lo != 0 && count >= (size_t(1) << 32))
            throw std::out_of_range("range sorts take fewer than 2^32 keys");
        enqueue_sort(ctx, keys, count, out, key_range, s, key_lo);
        ctx.pending = {true, s, count, key_range, false};
    });
}

bws_status bws_gpu_range_split(const uint32_t* keys, size_t count, uint64_t key_range, int parts,
                               uint32_t* out, uint32_t* d_counts, uint64_t* part_width, void* stream) {
    return wrap([&] {
        if (parts < 1 || parts > bws_gpu::MAX_BUCKETS) throw std::out_of_range("parts must be in [1, 4096]");
        if (key_range == 0 || key_range > kMaxKeyRange) throw std::out_of_range("key range must be in [1, 2^32]");
        if (d_counts == nullptr || part_width == nullptr || (count > 0 && (keys == nullptr || out == nullptr)))
            throw data_error("null pointer");
        if (count >= (size_t(1) << 32)) throw std::out_of_range("range split takes fewer than 2^32 keys");
        const bws_gpu::BucketPlan plan = bws_gpu::plan_range_split(key_range, parts);
        *part_width = plan.map.width == 0xffffffffu ? kMaxKeyRange : plan.map.width;
        const int dev = current_device();
        DeviceCtx& ctx = context_for(dev);
        std::lock_guard<std::mutex> lock(ctx.mu);
        ctx.init(dev);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        wait_done(ctx, s);
        preserve_pending(ctx, s);
        if (count == 0) {
            cuda_check(cudaMemsetAsync(d_counts, 0, sizeof(uint32_t) * parts, s), "count reset");
        } else {
            cuda_check(cudaMemsetAsync(ctx.ctrl_mem, 0, sizeof(Ctrl), s), "control block reset");
            int launches = 0;
            cuda_check(bws_gpu::launch_bucket_sort(keys, count, key_range, nullptr, out, ctx.bucket_scratch,
                                                   ctx.ctrl(), plan, ctx.geo, s, &launches, active_timer()),
                       "range split launch");
            g_launches.fetch_add(static_cast<uint64_t>(launches));
            cuda_check(cudaMemcpyAsync(d_counts, bws_gpu::bucket_totals(ctx.bucket_scratch, plan, ctx.geo),
                                       sizeof(uint32_t) * parts, cudaMemcpyDeviceToDevice, s),
                       "part counts");
            // keys >= key_range are counted by KB1: report them like a sort would
            unsigned int bad = 0;
            cuda_check(cudaMemcpyAsync(&bad, &ctx.ctrl()->bad_keys, sizeof(bad), cudaMemcpyDeviceToHost, s),
                       "bad key count");
            cuda_check(cudaStreamSynchronize(s), "range split execution");
            if (bad != 0)
                throw data_error(std::to_string(bad) + " key(s) not below the key range " +
                                 std::to_string(key_range));
        }
        record_done(ctx, s);
    });
}

bws_status bws_gpu_bitset_or_gather(const uint32_t* const* srcs, int nsrc, uint64_t n_words,
                                    uint32_t* dst, void* stream) {
    return wrap([&] {
        if (nsrc < 1 || nsrc > bws_gpu::MAX_OR_SOURCES) throw std::out_of_range("nsrc must be in [1, 8]");
        if (n_words > 0 && (srcs == nullptr || dst == nullptr)) throw data_error("null pointer");
        bws_gpu::OrSources os{};
        os.n = nsrc;
        for (int s = 0; s < nsrc; ++s) {
            if (n_words > 0 && srcs[s] == nullptr) throw data_error("null source pointer");
            os.p[s] = srcs[s];
        }
        const int dev = current_device();
        DeviceCtx& ctx = context_for(dev);
        std::lock_guard<std::mutex> lock(ctx.mu);
        ctx.init(dev);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        cuda_check(timed_launch("bitset_or_gather", s,
                                [&] { return bws_gpu::launch_or_gather(os, dst, n_words, ctx.geo, s); }),
                   "or_gather launch");
        g_launches.fetch_add(1);
    });
}

bws_status bws_gpu_ipc_get_handle(const void* dev_ptr, void* handle_out, uint64_t* offset_out) {
    return wrap([&] {
        if (dev_ptr == nullptr || handle_out == nullptr || offset_out == nullptr) throw data_error("null pointer");
        static_assert(sizeof(cudaIpcMemHandle_t) == BWS_GPU_IPC_HANDLE_BYTES, "IPC handle size");
        // the handle names the whole allocation (e.g. a caching allocator's
        // segment): report dev_ptr's offset inside it (driver entry point, so
        // the library needs no libcuda link)
        using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
        static GetRange get_range = [] {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q{};
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                fn = nullptr;
            return reinterpret_cast<GetRange>(fn);
        }();
        if (get_range == nullptr) throw std::runtime_error("cuMemGetAddressRange is unavailable");
        CUdeviceptr base = 0;
        size_t size = 0;
        if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
            throw std::runtime_error("cuMemGetAddressRange failed (not device memory?)");
        cudaIpcMemHandle_t h;
        cuda_check(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
        std::memcpy(handle_out, &h, sizeof(h));
        *offset_out = reinterpret_cast<uint64_t>(dev_ptr) - static_cast<uint64_t>(base);
    });
}

bws_status bws_gpu_ipc_open(const void* handle, void** dev_ptr_out) {
    return wrap([&] {
        if (handle == nullptr || dev_ptr_out == nullptr) throw data_error("null pointer");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        cuda_check(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle");
    });
}

bws_status bws_gpu_ipc_close(void* dev_ptr) {
    return wrap([&] { cuda_check(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle"); });
}

bws_status bws_gpu_sort_check(void* stream, uint64_t* distinct_out) {
    return wrap([&] {
        const int dev = current_device();
        DeviceCtx& ctx = context_for(dev);
        std::lock_guard<std::mutex> lock(ctx.mu);
        if (!ctx.ready || !ctx.pending.active) {
            if (distinct_out) *distinct_out = 0;
            return;
        }
        cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sort execution");
        cuda_check(cudaStreamSynchronize(ctx.pending.stream), "sort execution");
        Ctrl c;
        cuda_check(cudaMemcpy(&c, ctx.pending.snapped ? ctx.snap() : ctx.ctrl(), sizeof(Ctrl),
                              cudaMemcpyDeviceToHost),
                   "control block readback");
        const uint64_t range = ctx.pending.range ? ctx.pending.range : kMaxKeyRange;
        throw_bad_keys(c, range);
        if (c.total != ctx.pending.count)
            throw data_error("keys are not distinct: " + std::to_string(ctx.pending.count) + " keys, " +
                             std::to_string(c.total) + " distinct (the bitset sort requires distinct keys)");
        if (distinct_out) *distinct_out = c.total;
    });
}

bws_status bws_gpu_bitset_build(const uint32_t* keys, size_t count, uint32_t* bits,
                                uint64_t key_range, void* stream) {
    return wrap([&] {
        if (bits == nullptr || (count > 0 && keys == nullptr))
            throw data_error("null device pointer");
        check_range(key_range);
        if (key_range == 0) throw std::out_of_range("bitset_build needs a key range");
        const int dev = current_device();
        DeviceCtx& ctx = context_for(dev);
        std::lock_guard<std::mutex> lock(ctx.mu);
        ctx.init(dev);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const uint64_t words = (key_range + 31) / 32;
        wait_done(ctx, s);
        preserve_pending(ctx, s);
        cuda_check(cudaMemsetAsync(ctx.ctrl_mem, 0, sizeof(Ctrl), s), "control block reset");
        const int path = current_path();
        const bool bucketed = count < (size_t(1) << 32) &&
                              (path == BWS_PATH_BUCKETED || (path == BWS_PATH_AUTO && count >= kBucketedMinKeys));
        if (bucketed) {
            // KB1-KB3 + KB4b: SMEM-staged, coalesced, no atomics to global, no memset
            const bws_gpu::BucketPlan plan =
                bws_gpu::plan_buckets(key_range, ctx.geo.bucket_blocks[bws_gpu::MAX_BUCKET_SHIFT]);
            const size_t parted_cap = ctx.ensure_parted(count, plan);
            int launches = 0;
            cuda_check(bws_gpu::launch_bucket_sort(keys, count, key_range, nullptr, ctx.parted,
                                                   ctx.bucket_scratch, ctx.ctrl(), plan, ctx.geo, s,
                                                   &launches, active_timer(), bits, words, parted_cap),
                       "bucketed bitset build launch");
            g_launches.fetch_add(static_cast<uint64_t>(launches));
        } else {
            cuda_check(cudaMemsetAsync(bits, 0, words * sizeof(uint32_t), s), "bitset clear");
            cuda_check(timed_launch("bitset_scatter", s,
                                    [&] {
                                        return bws_gpu::launch_scatter(keys, count, bits, key_range,
                                                                       ctx.ctrl(), g_scatter_mode.load(),
                                                                       ctx.geo, s);
                                    }),
                       "bitset_scatter launch");
            g_launches.fetch_add(1);
        }
        record_done(ctx, s);
    });
}

bws_status bws_gpu_bitset_push(const uint32_t* keys, size_t count, uint64_t key_range, uint32_t* const* slices,
                               int nslices, uint64_t slice_words, void* stream) {
    return wrap([&] {
        if (nslices < 1 || nslices > bws_gpu::MAX_OR_SOURCES) throw std::out_of_range("nslices must be in [1, 8]");
        check_range(key_range);
        if (key_range == 0) throw std::out_of_range("bitset_push needs a key range");
        if (slice_words % 4 != 0) throw std::out_of_range("slice_words must be a multiple of 4");
        if (slice_words * static_cast<uint64_t>(nslices) < (key_range + 31) / 32)
            throw std::out_of_range("the slices do not cover the key range");
        if (count > 0 && keys == nullptr) throw data_error("null device pointer");
        if (count >= (size_t(1) << 32)) throw std::out_of_range("bitset_push takes fewer than 2^32 keys");
        bws_gpu::OrSources os{};
        os.n = nslices;
        for (int i = 0; i < nslices; ++i) {
            if (slices == nullptr || slices[i] == nullptr) throw data_error("null slice pointer");
            if (!bws_gpu::scan2_supported(slices[i])) throw data_error("slices must be 16-byte aligned");
            os.p[i] = slices[i];
        }
        if (count == 0) return;
        const int dev = current_device();
        DeviceCtx& ctx = context_for(dev);
        std::lock_guard<std::mutex> lock(ctx.mu);
        ctx.init(dev);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        wait_done(ctx, s);
        preserve_pending(ctx, s);
        cuda_check(cudaMemsetAsync(ctx.ctrl_mem, 0, sizeof(Ctrl), s), "control block reset");
        const bws_gpu::BucketPlan plan =
            bws_gpu::plan_buckets(key_range, ctx.geo.bucket_blocks[bws_gpu::MAX_BUCKET_SHIFT]);
        const size_t parted_cap = ctx.ensure_parted(count, plan);
        int launches = 0;
        cuda_check(bws_gpu::launch_bucket_push(keys, count, key_range, ctx.parted, ctx.bucket_scratch, ctx.ctrl(),
                                               plan, ctx.geo, s, &launches, os, slice_words, parted_cap,
                                               active_timer()),
                   "bitset push launch");
        g_launches.fetch_add(static_cast<uint64_t>(launches));
        record_done(ctx, s);
    });
}

bws_status bws_gpu_bitset_scan(const uint32_t* bits, uint64_t n_words, uint32_t key_base,
                               uint32_t* out, uint64_t out_capacity, uint64_t* d_total,
                               void* stream) {
    return wrap([&] {
        if (d_total == nullptr) throw data_error("null total pointer");
        if (n_words > 0 && (bits == nullptr || out == nullptr))
            throw data_error("null device pointer");
        if (n_words > kMaxWords) throw std::out_of_range("slice exceeds 2^27 words");
        const int dev = current_device();
        DeviceCtx& ctx = context_for(dev);
        std::lock_guard<std::mutex> lock(ctx.mu);
        ctx.init(dev);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (n_words == 0) {
            cuda_check(cudaMemsetAsync(d_total, 0, sizeof(uint64_t), s), "total reset");
            return;
        }
        const size_t tiles = bws_gpu::scan_tiles(n_words);
        wait_done(ctx, s);
        preserve_pending(ctx, s);
        cuda_check(cudaMemsetAsync(ctx.ctrl_mem, 0,
                                   sizeof(Ctrl) + tiles * sizeof(unsigned long long), s),
                   "control block reset");
        cuda_check(timed_launch("bitset_scan", s,
                                [&] {
                                    return launch_scan_any(
                                        bits, n_words, key_base, out, out_capacity, ctx.ctrl(),
                                        ctx.status(), reinterpret_cast<unsigned long long*>(d_total),
                                        /*clear=*/0, ctx.geo, s);
                                }),
                   "bitset_scan launch");
        g_launches.fetch_add(1);
        record_done(ctx, s);
    });
}

bws_status bws_gpu_bitset_scan_sources(const uint32_t* const* srcs, int nsrc, uint64_t n_words,
                                       uint32_t key_base, uint32_t* out, uint64_t out_capacity,
                                       uint64_t* d_total, void* stream) {
    return wrap([&] {
        if (nsrc < 1 || nsrc > bws_gpu::MAX_OR_SOURCES) throw std::out_of_range("nsrc must be in [1, 8]");
        if (d_total == nullptr) throw data_error("null total pointer");
        if (n_words > 0 && (srcs == nullptr || out == nullptr)) throw data_error("null device pointer");
        if (n_words > kMaxWords) throw std::out_of_range("slice exceeds 2^27 words");
        bws_gpu::OrSources os{};
        os.n = nsrc;
        bool aligned = true;
        for (int i = 0; i < nsrc; ++i) {
            if (n_words > 0 && srcs[i] == nullptr) throw data_error("null source pointer");
            os.p[i] = srcs[i];
            aligned &= bws_gpu::scan2_supported(srcs[i]);
        }
        const int dev = current_device();
        DeviceCtx& ctx = context_for(dev);
        std::lock_guard<std::mutex> lock(ctx.mu);
        ctx.init(dev);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (n_words == 0) {
            cuda_check(cudaMemsetAsync(d_total, 0, sizeof(uint64_t), s), "total reset");
            return;
        }
        const size_t tiles = bws_gpu::scan_tiles(n_words);
        wait_done(ctx, s);
        preserve_pending(ctx, s);
        cuda_check(cudaMemsetAsync(ctx.ctrl_mem, 0, sizeof(Ctrl) + tiles * sizeof(unsigned long long), s),
                   "control block reset");
        if (aligned) {
            // one kernel: the peers' words are ORed into the scan's SMEM tiles
            cuda_check(timed_launch("bitset_scan_sources", s,
                                    [&] {
                                        return bws_gpu::launch_scan2_sources(
                                            os, n_words, key_base, out, out_capacity, ctx.ctrl(),
                                            ctx.status(), reinterpret_cast<unsigned long long*>(d_total),
                                            ctx.geo, s);
                                    }),
                       "bitset_scan_sources launch");
            g_launches.fetch_add(1);
        } else {
            // a source not 16-byte aligned (no TMA / vector loads): OR-gather
            // into a stream-ordered temporary, then the plain scan
            void* tmp = nullptr;
            cuda_check(cudaMallocAsync(&tmp, n_words * sizeof(uint32_t), s), "slice allocation");
            uint32_t* slice = static_cast<uint32_t*>(tmp);
            cudaError_t err = timed_launch("bitset_or_gather", s, [&] {
                return bws_gpu::launch_or_gather(os, slice, n_words, ctx.geo, s);
            });
            if (err == cudaSuccess)
                err = timed_launch("bitset_scan", s, [&] {
                    return launch_scan_any(slice, n_words, key_base, out, out_capacity, ctx.ctrl(),
                                           ctx.status(), reinterpret_cast<unsigned long long*>(d_total),
                                           /*clear=*/0, ctx.geo, s);
                });
            cudaFreeAsync(tmp, s);
            cuda_check(err, "or_gather + bitset_scan launch");
            g_launches.fetch_add(2);
        }
        record_done(ctx, s);
    });
}

bws_status bws_gpu_set_scatter_mode(bws_scatter_mode mode) {
    return wrap([&] {
        if (mode < BWS_SCATTER_AUTO || mode > BWS_SCATTER_SMEM)
            throw config_error("unknown scatter mode");
        g_scatter_mode.store(static_cast<int>(mode));
    });
}

bws_status bws_gpu_set_path(bws_path path) {
    return wrap([&] {
        if (path < BWS_PATH_AUTO || path > BWS_PATH_SMALL) throw config_error("unknown path");
        g_path.store(static_cast<int>(path));
    });
}

uint64_t bws_gpu_launch_count(void) { return g_launches.load(); }

bws_status bws_gpu_set_kernel_timing(int enable) {
    return wrap([&] { g_timer.enabled.store(enable != 0); });
}

bws_status bws_gpu_kernel_timings(char* buf, size_t buf_size) {
    return wrap([&] {
        if (buf == nullptr || buf_size == 0) throw config_error("null output buffer");
        const std::string text = g_timer.collect();
        if (text.size() + 1 > buf_size)
            throw config_error("output buffer too small: need " + std::to_string(text.size() + 1) +
                               " bytes");
        std::memcpy(buf, text.c_str(), text.size() + 1);
    });
}

bws_status bws_gpu_set_device_count(int count) {
    return wrap([&] {
        if (count < 1) throw config_error("device count must be >= 1");
        std::vector<int> devs;
        if (count > 1)
            for (int i = 0; i < count; ++i) devs.push_back(i);
        multi_set_devices(devs);
    });
}

bws_status bws_gpu_set_devices(const int* devices, int count) {
    return wrap([&] {
        if (count < 1 || devices == nullptr) throw config_error("need at least one device");
        std::vector<int> devs(devices, devices + count);
        if (count == 1) devs.clear();  // one rank: the single-GPU path on the current device
        multi_set_devices(devs);
    });
}

int bws_gpu_device_count(void) {
    try {
        const int g = multi_rank_count();
        return g < 1 ? 1 : g;
    } catch (...) {
        return 1;
    }
}

void bws_gpu_shutdown(void) {
    multi_release();
    for (auto& ctx : g_ctx) {
        std::lock_guard<std::mutex> lock(ctx.mu);
        ctx.release();
    }
}

}  // extern "C"
