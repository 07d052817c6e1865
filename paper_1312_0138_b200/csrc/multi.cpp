// Single-process multi-GPU bitset sort behind the drop-in bws_sort (SURVEY.md
// §8(b) "bws_gpu_set_device_count / BITSORT_GPUS", §8(e), §3.5/§7.6).
//
// The reference's sort entry point (proj/include/bitsort/bitsort.h:89-90,
// called by proj/tools/main.cpp:127-144) takes one host array. With G > 1
// devices configured, a host-array bws_sort runs here, in the caller's
// process and thread, as the north star's partition:
//
//   1. shard      rank r takes keys [r n/G, (r+1) n/G) of the host array and
//                 copies them to its device over its own PCIe link (all G
//                 copies concurrently; pageable arrays through per-rank pinned
//                 bounce buffers, one host thread per rank)
//   2. range      no hint: K0 max per rank, M = max + 1 over ranks
//   3. build      every rank builds the FULL M-bit bitset of its shard
//                 (bucketed KB3 + KB4b for large shards, K2 for small ones)
//   4. exchange   NCCL: ncclReduceScatter(ncclUint32, ncclSum) inside one
//                 ncclGroupStart/End (exact: distinct keys set disjoint bits);
//                 rank r receives words [r W/G, (r+1) W/G), keys [r M/G, ...)
//                 P2P: no collective; rank r's scan reads word range r of
//                 every rank's bitset directly (peer access over NVLink, or
//                 plain loads when logical ranks share a device), ORed into
//                 the scan's shared-memory tiles (scan2 MULTI kernel)
//   5. scan       K3 over the slice -> c_r keys + the rank's count
//   6. offsets    the G counts to the host: offset_r = sum(c_<r); sum != n
//                 means repeated keys (data untouched, caller falls back)
//   7. write back rank r's c_r keys to data + offset_r (concurrently)
//
// NCCL is loaded with dlopen on first use (libnccl.so.2), so the library has
// no link-time dependency on it; ncclCommInitAll needs distinct devices, so
// logical ranks sharing a device (tests on one GPU) take the P2P exchange.
// Ordering between ranks uses CUDA events (cudaStreamWaitEvent across
// devices) and, for ranks sharing a device, the device context's `done`
// chain, which also serialises their use of its bucket buffers.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "host_internal.h"

namespace bws_host {
namespace {

// ---- NCCL through dlopen ----
struct NcclApi {
    bool tried = false;
    void* handle = nullptr;
    decltype(&ncclCommInitAll) comm_init_all = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclReduceScatter) reduce_scatter = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string why;

    bool load() {
        if (tried) return handle != nullptr;
        tried = true;
        const char* env = std::getenv("BITSORT_NCCL_LIB");
        for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
            if (!name) continue;
            handle = dlopen(name, RTLD_NOW | RTLD_LOCAL);
            if (handle) break;
        }
        if (!handle) {
            why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
            return false;
        }
        comm_init_all = reinterpret_cast<decltype(comm_init_all)>(dlsym(handle, "ncclCommInitAll"));
        comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(handle, "ncclCommDestroy"));
        reduce_scatter = reinterpret_cast<decltype(reduce_scatter)>(dlsym(handle, "ncclReduceScatter"));
        group_start = reinterpret_cast<decltype(group_start)>(dlsym(handle, "ncclGroupStart"));
        group_end = reinterpret_cast<decltype(group_end)>(dlsym(handle, "ncclGroupEnd"));
        error_string = reinterpret_cast<decltype(error_string)>(dlsym(handle, "ncclGetErrorString"));
        if (!comm_init_all || !comm_destroy || !reduce_scatter || !group_start || !group_end || !error_string) {
            why = "libnccl.so.2 lacks a required symbol";
            dlclose(handle);
            handle = nullptr;
            return false;
        }
        return true;
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess) throw internal_error(std::string(what) + ": " + error_string(r));
    }
};
NcclApi g_nccl;

// Per-logical-rank device resources (a device hosting several logical ranks
// holds one set per rank).
struct Rank {
    int dev = 0;
    cudaStream_t stream = nullptr;
    uint32_t* keys = nullptr;          // the rank's shard
    size_t keys_cap = 0;
    uint32_t* bits = nullptr;          // full bitset (padded to G * per words)
    size_t bits_cap = 0;
    uint32_t* slice = nullptr;         // NCCL: the reduce-scattered slice
    size_t slice_cap = 0;
    uint32_t* out = nullptr;           // sorted keys of the slice
    size_t out_cap = 0;
    unsigned char* ctrl_mem = nullptr; // Ctrl + scan tile status (kCtrlBytes)
    unsigned long long* d_count = nullptr;
    cudaEvent_t built = nullptr;
    void* bounce[2] = {nullptr, nullptr};  // pinned staging for pageable arrays
    cudaEvent_t bounce_ev[2] = {nullptr, nullptr};

    Ctrl* ctrl() { return reinterpret_cast<Ctrl*>(ctrl_mem); }
    unsigned long long* status() { return reinterpret_cast<unsigned long long*>(ctrl_mem + sizeof(Ctrl)); }
};

struct Multi {
    std::mutex mu;
    bool configured = false;
    std::vector<int> devices;  // logical rank -> device
    std::vector<Rank> ranks;
    std::vector<ncclComm_t> comms;
    bool peers_enabled = false;
};
Multi g_multi;

std::vector<int> parse_devices_env() {
    std::vector<int> devs;
    if (const char* e = std::getenv("BITSORT_DEVICES")) {  // explicit list, e.g. "0,0" (logical ranks)
        const char* p = e;
        while (*p) {
            char* end = nullptr;
            const long v = std::strtol(p, &end, 10);
            if (end == p) throw config_error(std::string("BITSORT_DEVICES: cannot parse '") + e + "'");
            devs.push_back(static_cast<int>(v));
            p = *end == ',' ? end + 1 : end;
        }
    } else if (const char* g = std::getenv("BITSORT_GPUS")) {
        const int n = std::atoi(g);
        if (n < 1) throw config_error(std::string("BITSORT_GPUS must be >= 1, got '") + g + "'");
        for (int i = 0; i < n; ++i) devs.push_back(i);
    }
    return devs;
}

void release_ranks(Multi& m) {
    for (size_t i = 0; i < m.comms.size(); ++i)
        if (m.comms[i]) g_nccl.comm_destroy(m.comms[i]);
    m.comms.clear();
    for (Rank& r : m.ranks) {
        cudaSetDevice(r.dev);
        if (r.stream) cudaStreamSynchronize(r.stream);
        cudaFree(r.keys);
        cudaFree(r.bits);
        cudaFree(r.slice);
        cudaFree(r.out);
        cudaFree(r.ctrl_mem);
        cudaFree(r.d_count);
        for (int i = 0; i < 2; ++i) {
            if (r.bounce[i]) cudaFreeHost(r.bounce[i]);
            if (r.bounce_ev[i]) cudaEventDestroy(r.bounce_ev[i]);
        }
        if (r.built) cudaEventDestroy(r.built);
        if (r.stream) cudaStreamDestroy(r.stream);
    }
    m.ranks.clear();
    m.peers_enabled = false;
}

void validate_devices(const std::vector<int>& devs) {
    const int visible = visible_devices();
    if (devs.empty() || devs.size() > static_cast<size_t>(bws_gpu::MAX_OR_SOURCES))
        throw config_error("multi-GPU sorts take 1 to " + std::to_string(bws_gpu::MAX_OR_SOURCES) +
                           " logical ranks, got " + std::to_string(devs.size()));
    for (int d : devs)
        if (d < 0 || d >= visible)
            throw config_error("device " + std::to_string(d) + " is not visible (" + std::to_string(visible) +
                               " CUDA device(s))");
}

// Caller holds m.mu.
void ensure_configured(Multi& m) {
    if (m.configured) return;
    std::vector<int> devs = parse_devices_env();
    if (!devs.empty()) validate_devices(devs);
    m.devices = devs;  // empty: single GPU
    m.configured = true;
}

bool all_distinct(const std::vector<int>& devs) {
    std::vector<int> s = devs;
    std::sort(s.begin(), s.end());
    return std::adjacent_find(s.begin(), s.end()) == s.end();
}

void ensure_ranks(Multi& m) {
    if (m.ranks.size() == m.devices.size()) return;
    release_ranks(m);
    m.ranks.resize(m.devices.size());
    for (size_t i = 0; i < m.devices.size(); ++i) {
        Rank& r = m.ranks[i];
        r.dev = m.devices[i];
        cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
        cuda_check(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaMalloc(&r.ctrl_mem, kCtrlBytes), "cudaMalloc(rank control block)");
        cuda_check(cudaMalloc(&r.d_count, sizeof(unsigned long long)), "cudaMalloc(rank count)");
        cuda_check(cudaEventCreateWithFlags(&r.built, cudaEventDisableTiming), "cudaEventCreate");
    }
}

template <class T>
T* grow(T*& p, size_t& cap, size_t n, const char* what) {
    if (n <= cap && p) return p;
    if (p) cuda_check(cudaFree(p), "cudaFree");
    p = nullptr;
    cap = 0;
    cuda_check(cudaMalloc(&p, std::max<size_t>(n, 4) * sizeof(T)), what);
    cap = std::max<size_t>(n, 4);
    return p;
}

// Host <-> rank copies of one shard: pinned arrays by one DMA each; pageable
// arrays in 16 MiB chunks through the rank's two pinned bounce buffers (the
// calling host thread's memcpy of chunk i+1 overlaps the DMA of chunk i).
void ensure_bounce(Rank& r) {
    if (r.bounce[0]) return;
    for (int i = 0; i < 2; ++i) {
        cuda_check(cudaHostAlloc(&r.bounce[i], kStageChunk, cudaHostAllocDefault), "cudaHostAlloc(staging)");
        cuda_check(cudaEventCreateWithFlags(&r.bounce_ev[i], cudaEventDisableTiming), "cudaEventCreate");
    }
}

void shard_to_device(Rank& r, const void* host, size_t bytes, bool pinned) {
    cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
    if (bytes == 0) return;
    if (pinned) {
        cuda_check(cudaMemcpyAsync(r.keys, host, bytes, cudaMemcpyHostToDevice, r.stream), "host-to-device copy");
        return;
    }
    ensure_bounce(r);
    for (size_t off = 0, i = 0; off < bytes; off += kStageChunk, ++i) {
        const int b = static_cast<int>(i & 1);
        const size_t len = std::min(kStageChunk, bytes - off);
        cuda_check(cudaEventSynchronize(r.bounce_ev[b]), "staging buffer reuse");
        std::memcpy(r.bounce[b], static_cast<const char*>(host) + off, len);
        cuda_check(cudaMemcpyAsync(reinterpret_cast<char*>(r.keys) + off, r.bounce[b], len, cudaMemcpyHostToDevice,
                                   r.stream),
                   "host-to-device copy");
        cuda_check(cudaEventRecord(r.bounce_ev[b], r.stream), "cudaEventRecord");
    }
}

void slice_to_host(Rank& r, void* host, size_t bytes, bool pinned) {
    cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
    if (bytes == 0) return;
    if (pinned) {
        cuda_check(cudaMemcpyAsync(host, r.out, bytes, cudaMemcpyDeviceToHost, r.stream), "device-to-host copy");
        cuda_check(cudaStreamSynchronize(r.stream), "device-to-host copy");
        return;
    }
    ensure_bounce(r);
    const size_t nch = (bytes + kStageChunk - 1) / kStageChunk;
    auto issue = [&](size_t i) {
        const int b = static_cast<int>(i & 1);
        const size_t off = i * kStageChunk;
        cuda_check(cudaMemcpyAsync(r.bounce[b], reinterpret_cast<const char*>(r.out) + off,
                                   std::min(kStageChunk, bytes - off), cudaMemcpyDeviceToHost, r.stream),
                   "device-to-host copy");
        cuda_check(cudaEventRecord(r.bounce_ev[b], r.stream), "cudaEventRecord");
    };
    for (size_t i = 0; i < nch && i < 2; ++i) issue(i);
    for (size_t i = 0; i < nch; ++i) {
        const int b = static_cast<int>(i & 1);
        const size_t off = i * kStageChunk;
        cuda_check(cudaEventSynchronize(r.bounce_ev[b]), "device-to-host copy");
        std::memcpy(static_cast<char*>(host) + off, r.bounce[b], std::min(kStageChunk, bytes - off));
        if (i + 2 < nch) issue(i + 2);
    }
}

// Runs f(rank index) for every rank on its own host thread (rank 0 on the
// caller's) and rethrows the first failure.
template <class F>
void for_each_rank_parallel(size_t G, F&& f) {
    std::vector<std::exception_ptr> errs(G);
    std::vector<std::thread> th;
    for (size_t g = 1; g < G; ++g)
        th.emplace_back([&, g] {
            try {
                f(g);
            } catch (...) {
                errs[g] = std::current_exception();
            }
        });
    try {
        f(0);
    } catch (...) {
        errs[0] = std::current_exception();
    }
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

enum class Exchange { Nccl, P2p };

Exchange pick_exchange(Multi& m) {
    int mode = 0;  // 0 auto, 1 nccl, 2 p2p
    if (const char* e = std::getenv("BITSORT_EXCHANGE")) {
        if (std::strcmp(e, "nccl") == 0) mode = 1;
        if (std::strcmp(e, "p2p") == 0) mode = 2;
    }
    const bool distinct = all_distinct(m.devices);
    if (mode == 2) return Exchange::P2p;
    if (mode == 1) {
        if (!distinct) throw config_error("the NCCL exchange needs distinct devices (ncclCommInitAll)");
        if (!g_nccl.load()) throw internal_error(g_nccl.why);
        return Exchange::Nccl;
    }
    return distinct && g_nccl.load() ? Exchange::Nccl : Exchange::P2p;
}

void ensure_comms(Multi& m) {
    if (!m.comms.empty()) return;
    m.comms.resize(m.devices.size(), nullptr);
    g_nccl.check(g_nccl.comm_init_all(m.comms.data(), static_cast<int>(m.devices.size()), m.devices.data()),
                 "ncclCommInitAll");
}

void ensure_peer_access(Multi& m) {
    if (m.peers_enabled) return;
    for (int a : m.devices)
        for (int b : m.devices) {
            if (a == b) continue;
            int can = 0;
            cuda_check(cudaDeviceCanAccessPeer(&can, a, b), "cudaDeviceCanAccessPeer");
            if (!can)
                throw internal_error("device " + std::to_string(a) + " cannot access device " + std::to_string(b) +
                                     " (the P2P exchange needs peer access; use BITSORT_EXCHANGE=nccl)");
            cuda_check(cudaSetDevice(a), "cudaSetDevice");
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "cudaDeviceEnablePeerAccess");
            cudaGetLastError();
        }
    m.peers_enabled = true;
}

}  // namespace

int multi_rank_count() {
    std::lock_guard<std::mutex> lock(g_multi.mu);
    ensure_configured(g_multi);
    return static_cast<int>(g_multi.devices.size());
}

void multi_set_devices(const std::vector<int>& devs) {
    std::lock_guard<std::mutex> lock(g_multi.mu);
    if (!devs.empty()) validate_devices(devs);
    if (g_multi.configured && devs == g_multi.devices) return;
    release_ranks(g_multi);
    g_multi.devices = devs;
    g_multi.configured = true;
}

std::vector<int> multi_devices() {
    std::lock_guard<std::mutex> lock(g_multi.mu);
    ensure_configured(g_multi);
    return g_multi.devices;
}

void multi_release() {
    std::lock_guard<std::mutex> lock(g_multi.mu);
    release_ranks(g_multi);
}

bool multi_sort_host(void* data, size_t count, uint64_t key_range) {
    NvtxRange nvtx_range("bitsort:multi-GPU bws_sort");
    Multi& m = g_multi;
    std::lock_guard<std::mutex> lock(m.mu);
    ensure_configured(m);
    const size_t G = m.devices.size();
    if (G < 2) throw internal_error("multi_sort_host needs >= 2 logical ranks");
    ensure_ranks(m);
    const Exchange ex = pick_exchange(m);
    if (ex == Exchange::Nccl) ensure_comms(m);
    if (ex == Exchange::P2p) ensure_peer_access(m);

    // every distinct device's context (bucket buffers, geometry), locked in
    // device order; ranks sharing a device are ordered by its `done` chain
    std::vector<int> devs = m.devices;
    std::sort(devs.begin(), devs.end());
    devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int d : devs) {
        DeviceCtx& ctx = context_for(d);
        locks.emplace_back(ctx.mu);
        ctx.init(d);
    }
    int prev = 0;
    cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    struct restore_device {
        int d;
        ~restore_device() { cudaSetDevice(d); }
    } restore{prev};

    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, data) != cudaSuccess) {
        cudaGetLastError();
        attr.type = cudaMemoryTypeUnregistered;
    }
    const bool pinned = attr.type == cudaMemoryTypeHost;
    uint32_t* host = static_cast<uint32_t*>(data);
    auto lo = [&](size_t g) { return count * g / G; };

    // 1. shards to their devices, concurrently
    for (size_t g = 0; g < G; ++g) {
        Rank& r = m.ranks[g];
        cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
        grow(r.keys, r.keys_cap, lo(g + 1) - lo(g), "cudaMalloc(rank keys)");
    }
    {
        NvtxRange nr("bitsort:multi-GPU host-to-device");
        for_each_rank_parallel(G, [&](size_t g) {
            shard_to_device(m.ranks[g], host + lo(g), (lo(g + 1) - lo(g)) * sizeof(uint32_t), pinned);
        });
    }

    // 2. key range: the max over the ranks' K0 when there is no hint
    const bool check_bad = key_range != 0 && key_range < kMaxKeyRange;
    if (key_range == 0) {
        for (size_t g = 0; g < G; ++g) {
            Rank& r = m.ranks[g];
            cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
            cuda_check(cudaMemsetAsync(r.ctrl_mem, 0, sizeof(Ctrl), r.stream), "control block reset");
            if (lo(g + 1) > lo(g)) {
                cuda_check(bws_gpu::launch_key_max(r.keys, lo(g + 1) - lo(g), r.ctrl(), context_for(r.dev).geo,
                                                   r.stream, 0),
                           "key_max launch");
                g_launches.fetch_add(1);
            }
        }
        uint32_t mx = 0;
        for (size_t g = 0; g < G; ++g) {
            Rank& r = m.ranks[g];
            Ctrl c;
            cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
            cuda_check(cudaMemcpyAsync(&c, r.ctrl(), sizeof(Ctrl), cudaMemcpyDeviceToHost, r.stream), "max readback");
            cuda_check(cudaStreamSynchronize(r.stream), "key_max execution");
            mx = std::max(mx, c.max_key);
        }
        key_range = static_cast<uint64_t>(mx) + 1;
    }
    const uint64_t words = (key_range + 31) / 32;
    const uint64_t per = ((words + G - 1) / G + 3) & ~uint64_t(3);  // whole 16-byte units per rank
    const uint64_t words_pad = per * G;

    // 3. every rank builds the full bitset of its shard
    for (size_t g = 0; g < G; ++g) {
        Rank& r = m.ranks[g];
        DeviceCtx& ctx = context_for(r.dev);
        const size_t n_g = lo(g + 1) - lo(g);
        cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
        grow(r.bits, r.bits_cap, words_pad, "cudaMalloc(rank bitset)");
        wait_done(ctx, r.stream);
        preserve_pending(ctx, r.stream);
        cuda_check(cudaMemsetAsync(r.ctrl_mem, 0, sizeof(Ctrl), r.stream), "control block reset");
        if (words_pad > words)
            cuda_check(cudaMemsetAsync(r.bits + words, 0, (words_pad - words) * sizeof(uint32_t), r.stream),
                       "bitset padding");
        const int path = current_path();
        const bool bucketed = n_g < (size_t(1) << 32) &&
                              (path == BWS_PATH_BUCKETED || (path == BWS_PATH_AUTO && n_g >= kBucketedMinKeys));
        if (n_g == 0) {
            cuda_check(cudaMemsetAsync(r.bits, 0, words * sizeof(uint32_t), r.stream), "bitset clear");
        } else if (bucketed) {
            const bws_gpu::BucketPlan plan =
                bws_gpu::plan_buckets(key_range, ctx.geo.bucket_blocks[bws_gpu::MAX_BUCKET_SHIFT]);
            const size_t parted_cap = ctx.ensure_parted(n_g, plan);
            int launches = 0;
            cuda_check(bws_gpu::launch_bucket_sort(r.keys, n_g, key_range, nullptr, ctx.parted, ctx.bucket_scratch,
                                                   r.ctrl(), plan, ctx.geo, r.stream, &launches, active_timer(),
                                                   r.bits, words, parted_cap),
                       "bucketed bitset build launch");
            g_launches.fetch_add(static_cast<uint64_t>(launches));
        } else {
            cuda_check(cudaMemsetAsync(r.bits, 0, words * sizeof(uint32_t), r.stream), "bitset clear");
            cuda_check(timed_launch("bitset_scatter", r.stream,
                                    [&] {
                                        return bws_gpu::launch_scatter(r.keys, n_g, r.bits, key_range, r.ctrl(),
                                                                       g_scatter_mode.load(), ctx.geo, r.stream);
                                    }),
                       "bitset_scatter launch");
            g_launches.fetch_add(1);
        }
        record_done(ctx, r.stream);
        cuda_check(cudaEventRecord(r.built, r.stream), "cudaEventRecord");
    }
    uint64_t bad = 0;
    if (check_bad) {
        for (size_t g = 0; g < G; ++g) {
            Rank& r = m.ranks[g];
            unsigned int b = 0;
            cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
            cuda_check(cudaMemcpyAsync(&b, &r.ctrl()->bad_keys, sizeof(b), cudaMemcpyDeviceToHost, r.stream),
                       "bad key count");
            cuda_check(cudaStreamSynchronize(r.stream), "bitset build");
            bad += b;
        }
        if (bad) throw data_error(std::to_string(bad) + " key(s) not below the key range " + std::to_string(key_range));
    }

    // 4 + 5. exchange, then each rank scans its slice
    auto capacity = [&](size_t g) {
        const uint64_t klo = g * per * 32;
        const uint64_t khi = std::min<uint64_t>((g + 1) * per * 32, key_range);
        return static_cast<size_t>(khi > klo ? std::min<uint64_t>(count, khi - klo) : 0);
    };
    for (size_t g = 0; g < G; ++g) {
        Rank& r = m.ranks[g];
        cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
        grow(r.out, r.out_cap, capacity(g), "cudaMalloc(rank output)");
        if (ex == Exchange::Nccl) grow(r.slice, r.slice_cap, per, "cudaMalloc(rank slice)");
    }
    if (ex == Exchange::Nccl) {
        NvtxRange nr("bitsort:NCCL reduce-scatter");
        g_nccl.check(g_nccl.group_start(), "ncclGroupStart");
        for (size_t g = 0; g < G; ++g) {
            Rank& r = m.ranks[g];
            cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
            g_nccl.check(g_nccl.reduce_scatter(r.bits, r.slice, per, ncclUint32, ncclSum, m.comms[g], r.stream),
                         "ncclReduceScatter");
        }
        g_nccl.check(g_nccl.group_end(), "ncclGroupEnd");
    }
    for (size_t g = 0; g < G; ++g) {
        Rank& r = m.ranks[g];
        DeviceCtx& ctx = context_for(r.dev);
        cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
        const uint32_t key_base = static_cast<uint32_t>(g * per * 32);
        cuda_check(cudaMemsetAsync(r.ctrl_mem, 0, sizeof(Ctrl) + bws_gpu::scan_tiles(per) * 4 * sizeof(unsigned long long),
                                   r.stream),
                   "control block reset");
        if (ex == Exchange::Nccl) {
            cuda_check(timed_launch("bitset_scan", r.stream,
                                    [&] {
                                        return launch_scan_any(r.slice, per, key_base, r.out, capacity(g), r.ctrl(),
                                                               r.status(), r.d_count, /*clear=*/0, ctx.geo, r.stream);
                                    }),
                       "bitset_scan launch");
            g_launches.fetch_add(1);
        } else {
            NvtxRange nr("bitsort:P2P scan over the ranks' bitsets");
            bws_gpu::OrSources os{};
            os.n = static_cast<int>(G);
            os.p[0] = r.bits + g * per;  // the local words first (TMA), peers by 16-byte loads
            int k = 1;
            for (size_t h = 0; h < G; ++h) {
                if (h == g) continue;
                cuda_check(cudaStreamWaitEvent(r.stream, m.ranks[h].built, 0), "cross-rank ordering");
                os.p[k++] = m.ranks[h].bits + g * per;
            }
            cuda_check(timed_launch("bitset_scan_sources", r.stream,
                                    [&] {
                                        return bws_gpu::launch_scan2_sources(os, per, key_base, r.out, capacity(g),
                                                                             r.ctrl(), r.status(), r.d_count, ctx.geo,
                                                                             r.stream);
                                    }),
                       "bitset_scan_sources launch");
            g_launches.fetch_add(1);
        }
    }

    // 6. counts -> offsets; repeated keys lower the total
    std::vector<unsigned long long> cnt(G, 0);
    for (size_t g = 0; g < G; ++g) {
        Rank& r = m.ranks[g];
        cuda_check(cudaSetDevice(r.dev), "cudaSetDevice");
        cuda_check(cudaMemcpyAsync(&cnt[g], r.d_count, sizeof(unsigned long long), cudaMemcpyDeviceToHost, r.stream),
                   "count readback");
    }
    uint64_t total = 0;
    for (size_t g = 0; g < G; ++g) {
        cuda_check(cudaSetDevice(m.ranks[g].dev), "cudaSetDevice");
        cuda_check(cudaStreamSynchronize(m.ranks[g].stream), "multi-GPU sort");
        total += cnt[g];
    }
    if (total != count) return false;

    // 7. every rank's slice to its place in the host array, concurrently
    {
        NvtxRange nr("bitsort:multi-GPU device-to-host");
        std::vector<size_t> off(G, 0);
        for (size_t g = 1; g < G; ++g) off[g] = off[g - 1] + cnt[g - 1];
        for_each_rank_parallel(G, [&](size_t g) {
            slice_to_host(m.ranks[g], host + off[g], cnt[g] * sizeof(uint32_t), pinned);
        });
    }
    return true;
}

}  // namespace bws_host
