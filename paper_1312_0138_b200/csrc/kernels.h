// Launch interface of the sm_100a bitset-sort kernels (K2 scatter, K3 scan)
// and the per-sort control block they share. Host orchestration lives in
// capi.cpp; nothing here is exported from libbitsort.so.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace bws_gpu {

// Per-sort device control block. Zeroed (cudaMemsetAsync) before every sort
// together with the scan's tile-status array, which directly follows it.
struct alignas(64) Ctrl {
    unsigned int max_key;          // atomicMax over every in-range key (K2)
    unsigned int bad_keys;         // keys >= key_range (K2); never scattered
    unsigned int ticket;           // K3 dynamic tile ticket / KB4 bucket ticket
    unsigned int done_ctas;        // slab KB3: CTAs finished (the last one scans the counts)
    unsigned long long total;      // set bits over the whole scan (K3, last tile)
    unsigned int min_inv;          // ~(min key), atomicMax (K0): zero-initialised like max_key
    unsigned int error;            // KF: ring protocol timeout (the ring state is then reset)
    unsigned int overflow;         // slab KB3: a bucket's runs were dropped (repeated keys)
    unsigned int pad2;
    unsigned long long pad1[3];
};
static_assert(sizeof(Ctrl) == 64, "Ctrl is one 64-byte line");

// K3 geometry: a tile is SCAN_ROUNDS rounds of SCAN_THREADS consecutive words.
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ROUNDS = 8;
constexpr int SCAN_TILE_WORDS = SCAN_THREADS * SCAN_ROUNDS;  // 2048 words = 65536 keys

// K3 v2 geometry (scan.cu): 8192-word tiles via TMA, 16 warps, 2 CTAs/SM.
constexpr int SCAN2_THREADS = 512;
constexpr int SCAN2_TILE_WORDS = 8192;
constexpr int SCAN2_STAGE = 640;  // keys per warp stage
constexpr std::size_t scan2_smem_bytes() {
    return 2 * SCAN2_TILE_WORDS * 4 + (SCAN2_THREADS / 32) * (SCAN2_STAGE + SCAN2_STAGE / 32) * 4;  // 2nd buffer spare
}

// K2 geometry: a tile is SCATTER_VEC uint4 loads per thread.
constexpr int SCATTER_THREADS = 256;
constexpr int SCATTER_VEC = 4;
constexpr int SCATTER_TILE_KEYS = SCATTER_THREADS * SCATTER_VEC * 4;  // 4096 keys
constexpr int SCATTER_SMEM_WORDS = 8192;  // staged bitset window: 32 KB = 262144 keys

enum ScatterMode : int { kAuto = 0, kPlain = 1, kWarpAgg = 2, kSmem = 3 };

inline std::size_t scan_tiles(std::uint64_t n_words) {
    return static_cast<std::size_t>((n_words + SCAN_TILE_WORDS - 1) / SCAN_TILE_WORDS);
}

// Bucketed pipeline geometry (bucket.cu).
constexpr int MAX_BUCKETS = 4096;
constexpr int MIN_BUCKET_SHIFT = 15;  // SMEM bitset of a bucket: 2^shift bits
constexpr int MAX_BUCKET_SHIFT = 20;  // 128 KB
constexpr int BUCKET_HIST_THREADS = 512;
constexpr int HIST_SPLIT = 4;  // histogram CTAs per partition CTA share
// KB3 variants: "wide" (nb <= 4096): 1024 threads, 16384-key tiles, 1 CTA/SM;
// "narrow" (nb <= 1024): 512 threads, 8192-key tiles, 2 CTAs/SM.
constexpr int PART_THREADS = 1024;
constexpr int PART_KPT = 16;
constexpr int PART_TILE = PART_THREADS * PART_KPT;  // 16384 keys per wide tile
constexpr int PART_NARROW_THREADS = 512;
constexpr int PART_NARROW_MAXB = 1024;
constexpr int BUCKET_THREADS = 1024;
constexpr int BUCKET_STAGE = 640;        // keys per warp in the extraction stage (2^20 buckets)

constexpr int PART_KPT_SLAB = 20;   // slab KB3 with <= 1024 buckets: 20480-key tiles
constexpr int PART_DUMP = 32768;    // slab overflow tile (>= any KB3 tile)
constexpr std::size_t part_smem_bytes(int threads, int maxb, int kpt = PART_KPT) {
    return 2 * std::size_t(threads) * kpt * 4 + std::size_t(maxb + 1) * 16;  // TMA ring + 4 slot arrays
}
// KB4 CTA shape per bucket class: 2^20-bit buckets (128 KB bitset) one
// 1024-thread CTA per SM; narrower buckets 512-thread CTAs, two per SM, so
// one CTA's scatter (HBM reads) overlaps the other's extraction.
constexpr int bucket_sort_threads(int shift) { return shift >= MAX_BUCKET_SHIFT ? BUCKET_THREADS : 512; }
constexpr std::size_t bucket_sort_smem_bytes(int shift) {
    return (std::size_t(1) << (shift - 3)) + (std::size_t(1) << (shift - 8)) +  // bitset + summary
           (bucket_sort_threads(shift) / 32) * (BUCKET_STAGE + BUCKET_STAGE / 32) * 4;
}


struct LaunchGeometry {
    int scatter_blocks = 0;
    int scan_blocks = 0;
    int fill_blocks = 0;
    int part_blocks = 0;                         // KB1/KB3 shares, wide KB3 variant
    int part_blocks_narrow = 0;                  // KB1/KB3 shares, narrow KB3 variant
    int bucket_blocks[MAX_BUCKET_SHIFT + 1] = {};  // KB4 CTAs per bucket shift
    int scan2_blocks = 0;                          // K3 v2 CTAs
    int multiset_blocks = 0;                       // KB4m CTAs (one per SM)
    int fused_ctas = 0;                            // KF CTAs (one per SM; 0: no cooperative launch)
    std::size_t fused_smem_limit = 0;              // KF dynamic SMEM ceiling
    int small_ctas = 0;                            // KS CTAs (one per SM; 0: no cooperative launch)
};

// A key array as seen by the bucketed kernels: 16-byte-aligned uint4 body plus
// up to 3 misaligned head and 3 tail keys.
struct KeySplit {
    const uint4* body = nullptr;
    std::size_t nv = 0;
    const std::uint32_t* head = nullptr;
    int n_head = 0;
    const std::uint32_t* tail = nullptr;
    int n_tail = 0;
    std::uint32_t xr = 0;  // keys are XORed with this on load (signed int32: 0x80000000 maps
                           // the signed order onto the unsigned one)
};

// Bucket of a key: floor(key / width), width = q * 2^ms with q <= 8, computed
// as __umulhi((key >> ms) << 12, mq), mq = ceil(2^20 / q). Exact for every
// uint32 key: the pre-shifted key is < 2^17 (ms >= 15), so the rounding error
// of mq stays below one bucket step.
struct BucketMap {
    int ms = 20;
    std::uint32_t mq = 1u << 20;
    std::uint32_t width = 1u << 20;  // keys per bucket
    std::uint32_t lo = 0;            // first key of bucket 0 (range sorts); key - lo is bucketed
    std::uint32_t xr = 0;            // output keys are XORed with this (signed sorts: 0x80000000)
};

struct BucketPlan {
    int shift = 20;   // SMEM bitset class of a bucket: 2^shift bits >= map.width
    int nb = 1;       // number of buckets, <= MAX_BUCKETS
    BucketMap map;
    bool partition_only = false;  // stop after KB3 (range split: packed groups, totals in scratch)
};

// Slab layout of the bucket buffer (KB3 without KB1/KB2): bucket b owns the
// fixed slots [b * cap, (b + 1) * cap), cap = min(2^shift, n) rounded up to 4,
// which no set of DISTINCT keys can overflow; per-bucket fill counters replace
// the histogram pass. A claim that repeated keys push past a bucket's
// capacity is aimed at `dump` (past the last bucket) and its stores are
// skipped: that bucket then sorts nothing, so the popcount total reports the
// repeats.
struct SlabArgs {
    std::uint32_t* gcnt = nullptr;         // nb zeroed fill counters
    std::uint32_t cap = 0;                 // slots per bucket
    std::uint32_t dump = 0;                // nb * cap: claims at or past it are overflow (dropped)
    std::uint32_t limit = 0;               // keys >= limit are counted as bad (check != 0)
    int check = 0;
    Ctrl* ctrl = nullptr;
    std::uint32_t* tot = nullptr;          // out: keys per bucket (slots to read, padding included)
    unsigned long long* g_base = nullptr;  // out: output offset per bucket (+ total at [nb])
    std::uint32_t* gtrue = nullptr;        // TMA-store KB3: true keys per bucket (gcnt counts
                                           // slots, padded to multiples of 4); zeroed like gcnt
    std::uint32_t* order = nullptr;        // packed KB3 (CTA 0): KB4 ticket order, largest
                                           // buckets first; order[nb] = 0 means identity
    std::uint32_t* chunk_tab = nullptr;    // chunked layout: nb x max_chunks pool chunk ids + 1 (zeroed)
    std::uint32_t max_chunks = 0;
    std::uint32_t* pool_next = nullptr;    // chunked layout: next free pool chunk - nb (zeroed)
    std::uint32_t chunk_shift = 13;        // chunked layout: log2 slots per pool chunk
    std::uint32_t chunk_pad = 0;           // chunked layout: pool chunk id starts at slot id * (2^shift + pad)
                                           // (a multiple of 4): chunk starts off the power-of-two stride
};
constexpr std::uint32_t KC_CHUNK_MIN = 8192;      // smallest pool chunk (chunked layout)
constexpr std::uint32_t KC_DROP = 0xffffffffu;    // a dropped (overflowed) run

// Optional per-kernel timing hook (bench.py's live roofline): before() and
// after() bracket every kernel launch on the launching stream.
struct KernelTimer {
    virtual void before(cudaStream_t stream) = 0;
    virtual void after(const char* kernel, cudaStream_t stream) = 0;
    virtual ~KernelTimer() = default;
};

// Computes persistent-grid sizes (SM count x resident blocks) for `device`.
cudaError_t query_geometry(int device, LaunchGeometry* geo);

// K2: bits[x>>5] |= 1<<(x&31) for every key x < key_range (key_range in
// [1, 2^32]); keys >= key_range are counted in ctrl->bad_keys. Also folds the
// max in-range key into ctrl->max_key.
cudaError_t launch_scatter(const std::uint32_t* keys, std::size_t n, std::uint32_t* bits,
                           std::uint64_t key_range, Ctrl* ctrl, int mode,
                           const LaunchGeometry& geo, cudaStream_t stream);

// K3: single-pass decoupled-lookback scan of n_words words (n_words == 0:
// (ctrl->max_key >> 5) + 1, i.e. derived from K2). Writes key_base + bit index
// of every set bit, ascending, to out[0, out_capacity). Writes the number of
// set bits to ctrl->total and, if non-null, *d_total. With clear != 0 every
// nonzero word is zeroed after it is read (keeps a cached bitset all-zero
// between sorts). `status` holds scan_tiles(n_words) zeroed 64-bit words.
cudaError_t launch_scan(const std::uint32_t* bits, std::uint64_t n_words, std::uint32_t key_base,
                        std::uint32_t* out, std::uint64_t out_capacity, Ctrl* ctrl,
                        unsigned long long* status, unsigned long long* d_total, int clear,
                        const LaunchGeometry& geo, cudaStream_t stream);

// K3 v2 (scan.cu): same contract as launch_scan; needs a 16-byte-aligned
// bitset (scan2_supported). status needs ceil(n_words / 8192) zeroed words.
bool scan2_supported(const std::uint32_t* bits);
cudaError_t configure_scan2(int device, LaunchGeometry* geo);
// two_pass: tile popcounts + their prefix first (no lookback; needs
// n_words > 0 known on the host), then the same extraction.
cudaError_t launch_scan2(std::uint32_t* bits, std::uint64_t n_words, std::uint32_t key_base,
                         std::uint32_t* out, std::uint64_t out_capacity, Ctrl* ctrl,
                         unsigned long long* status, unsigned long long* d_total, int clear,
                         const LaunchGeometry& geo, cudaStream_t stream, int two_pass,
                         int* launches);

// Bucketed pipeline (bucket.cu). plan_buckets picks the bucket width for a
// key range; bucket_scratch_bytes sizes the histogram/offset scratch.
// Range split into `parts` groups of consecutive key ranges (multi-GPU key
// all-to-all): group width = the smallest q * 2^s >= ceil(key_range / parts)
// (q <= 8, s >= 12), so the bucket map stays exact; the last group is shorter.
BucketPlan plan_range_split(std::uint64_t key_range, int parts);
// Bucket totals (uint32 per bucket) in the scratch of the last launch_bucket_sort.
const std::uint32_t* bucket_totals(const void* scratch, const BucketPlan& plan, const LaunchGeometry& geo);
// kb4_ctas: resident KB4 CTAs (0: power-of-two widths only).
BucketPlan plan_buckets(std::uint64_t key_range, int kb4_ctas);
// Bucket plan of the multiset (repeated keys) pass: the narrowest power-of-two
// buckets with at most MAX_BUCKETS of them.
BucketPlan plan_multiset(std::uint64_t key_range);
// Bucket-buffer slots the slab layout needs for n keys (0: use the packed
// histogram layout: the slab would exceed 4n slots or 2^32).
std::uint64_t slab_slots(const BucketPlan& plan, std::size_t n);
// Pool slots the chunked layout needs for n keys (0: disabled, BITSORT_CHUNK=0).
std::uint64_t chunk_slots(const BucketPlan& plan, std::size_t n);
std::size_t bucket_scratch_bytes(const BucketPlan& plan, int hist_blocks);
cudaError_t configure_bucket_kernels(int device, LaunchGeometry* geo);
// KB1..KB4: sorts n keys (all < key_range) into out via the `parted` buffer
// of parted_cap slots (>= n; the slab layout is used when parted_cap >=
// slab_slots(plan, n) > 0, and then KB1/KB2 are skipped). Adds the number of
// distinct keys to ctrl->total, counts keys >= key_range in ctrl->bad_keys.
// `launches` receives the kernel count. With bits_out set, KB4b writes the
// bitset (n_words words) instead of sorted keys (multi-GPU per-rank build; no
// clearing of bits_out needed). With multiset, repeated keys are sorted too
// (packed layout + KB4m per-bucket counting sort; ctrl->total counts every
// key written): bws_sort on inputs that are not distinct.
cudaError_t launch_bucket_sort(const std::uint32_t* keys, std::size_t n, std::uint64_t key_range,
                               std::uint32_t* out, std::uint32_t* parted, void* scratch, Ctrl* ctrl,
                               const BucketPlan& plan, const LaunchGeometry& geo,
                               cudaStream_t stream, int* launches, KernelTimer* timer = nullptr,
                               std::uint32_t* bits_out = nullptr, std::uint64_t n_words = 0,
                               std::uint64_t parted_cap = 0, bool multiset = false,
                               const struct OrSources* push = nullptr, std::uint64_t push_slice_words = 0,
                               int inplace_mode = 0);
// inplace_mode (slab layout only, out == keys): 1 = KB4 writes nothing if any
// bucket's runs were dropped (ctrl->overflow: the keys stay intact for the
// counting pass); 2 = recovery after a mode-1 sort found repeats without
// overflow: KB4m counting-sorts every bucket from the slabs the mode-1 KB3
// left (same keys, plan and buffers; ctrl ticket/total zeroed by the caller).
// slab_in_use: whether launch_bucket_sort takes the slab layout for (plan, n).
bool slab_in_use(const BucketPlan& plan, std::size_t n, std::uint64_t parted_cap);
// Multi-GPU OR-gather (the P2P replacement of the reduce-scatter): dst[i] =
// OR over s of srcs.p[s][i] for i < n_words; srcs may point into peer GPUs'
// memory (CUDA IPC over NVLink/NVSwitch).
constexpr int MAX_OR_SOURCES = 8;
struct OrSources {
    const std::uint32_t* p[MAX_OR_SOURCES];
    int n;
};
cudaError_t launch_or_gather(const OrSources& srcs, std::uint32_t* dst, std::uint64_t n_words,
                             const LaunchGeometry& geo, cudaStream_t stream);
// Multi-GPU push build (the exchange fused into the build): KB1-KB3, then
// KB4p ORs every bucket's SMEM bitset straight into the owner rank's slice
// (slices.p[r] covers words [r * slice_words, (r + 1) * slice_words), 16-byte
// aligned, zeroed by the owner beforehand; slice_words a multiple of 4) with
// bulk OR-reductions; peers' slices are CUDA IPC pointers over NVLink.
cudaError_t launch_bucket_push(const std::uint32_t* keys, std::size_t n, std::uint64_t key_range,
                               std::uint32_t* parted, void* scratch, Ctrl* ctrl, const BucketPlan& plan,
                               const LaunchGeometry& geo, cudaStream_t stream, int* launches,
                               const OrSources& slices, std::uint64_t slice_words, std::uint64_t parted_cap,
                               KernelTimer* timer = nullptr);
// K3 v2 over the OR of srcs (the fused P2P exchange + scan): same contract as
// launch_scan2 (lookback variant, no clearing) on the virtual bitset
// OR_s srcs.p[s][0, n_words); every source 16-byte aligned (scan2_supported).
// srcs.p[0] (the local slice) arrives by TMA, peers by 16-byte loads.
cudaError_t launch_scan2_sources(const OrSources& srcs, std::uint64_t n_words, std::uint32_t key_base,
                                 std::uint32_t* out, std::uint64_t out_capacity, Ctrl* ctrl,
                                 unsigned long long* status, unsigned long long* d_total,
                                 const LaunchGeometry& geo, cudaStream_t stream);
// Other widths (widths.cu). 8/16-bit keys: counting sort over the type's
// whole range, in place on device memory (scratch: width_scratch_bytes()).
std::size_t width_scratch_bytes();
cudaError_t configure_width_kernels(int device, LaunchGeometry* geo);
cudaError_t launch_sort_small(void* data, std::size_t n, int width, int is_unsigned, void* scratch,
                              const LaunchGeometry& geo, cudaStream_t stream, int* launches,
                              KernelTimer* timer = nullptr);
// 64-bit keys: (min, max) of the biased keys into scratch[0..1] (u64), then
// narrowing to u32 offsets from the min and widening back (scratch holds the min).
cudaError_t launch_minmax64(const std::uint64_t* keys, std::size_t n, int is_unsigned, void* scratch,
                            const LaunchGeometry& geo, cudaStream_t stream);
cudaError_t launch_narrow64(const std::uint64_t* keys, std::size_t n, int is_unsigned, const void* scratch,
                            std::uint32_t* out, const LaunchGeometry& geo, cudaStream_t stream);
cudaError_t launch_widen64(const std::uint32_t* sorted, std::size_t n, int is_unsigned, const void* scratch,
                           std::uint64_t* out, const LaunchGeometry& geo, cudaStream_t stream);
// 64-bit keys of any span: stable LSD radix sort with 8-bit digits. hist:
// scratch[0 .. 8*256) u64 = global histogram of every digit of the biased
// keys (the host skips digits on which all keys agree); pass: one stable
// scatter by digit `digit` from in to out (keys XORed with xin on load and
// xout on store, n < 2^32).
std::size_t radix64_scratch_bytes(const LaunchGeometry& geo);
cudaError_t launch_radix64_hist(const std::uint64_t* keys, std::size_t n, int is_unsigned, void* scratch,
                                const LaunchGeometry& geo, cudaStream_t stream);
cudaError_t launch_radix64_pass(const std::uint64_t* in, std::uint64_t* out, std::size_t n, int digit,
                                std::uint64_t xin, std::uint64_t xout, void* scratch, const LaunchGeometry& geo,
                                cudaStream_t stream);
// KF (fused.cu): the whole sort in one persistent cooperative kernel, the
// bitset of a pass split into per-SM slices held in shared memory, keys moved
// to their slice's SM through L2-resident per-owner rings. For key ranges
// whose bitset fits in <= 2 passes (plan_fused().ok).
constexpr int KF_MAXG = 192;  // owners (CTAs = SMs) the state is sized for
struct FusedPlan {
    bool ok = false;
    int P = 1;                 // passes over the keys
    int G = 0;                 // CTAs = owners
    std::uint32_t S = 0;       // slice bits per owner (multiple of 2^17)
    std::uint32_t H = 0;       // G * S: keys [p H, (p + 1) H) in pass p (P == 2)
    std::uint32_t mag = 0;     // ceil(2^32 / (S >> 12)): owner = umulhi(x >> 12, mag)
    std::size_t smem = 0;      // dynamic SMEM per CTA
};
struct FusedArgs {
    KeySplit ks;
    std::uint32_t range_m1;    // keys x with (x ^ xr) - lo > range_m1 are bad
    std::uint32_t lo;
    std::uint32_t H, S, mag;
    int P;
    std::uint32_t* out;
    Ctrl* ctrl;                // total, bad_keys, error = protocol timeout (written by CTA 0)
    std::uint32_t* rings;      // 2 sets x G owners x 8 sub-rings of 2^12 entries
    std::uint32_t* tail;       // claim counter per sub-ring
    std::uint32_t* head;       // consumed counter per sub-ring
    std::uint32_t* sync;       // done[0], done[1], CTAs out, error
    unsigned long long* counts;// 3 x G published counts (flag bit 63)
    std::uint32_t* saved;      // G x S/32 words: pass-0 slices (P == 2)
    unsigned long long* trace; // optional: per CTA phase timestamps + spin counts (9 words)
    std::uint32_t* gbits;      // direct mode (KD, P == 1): the all-zero global bitset, >= G * S bits;
                               // keys are ORed into it, then each CTA takes (and zeroes) its slice
};
FusedPlan plan_fused(std::uint64_t key_range, int sms, std::size_t smem_limit);
std::size_t fused_state_bytes(int sms);
cudaError_t configure_fused(int device, LaunchGeometry* geo);
// (Re)initialises the persistent ring state (rings to 0xFF, counters to 0).
cudaError_t init_fused_state(void* state, int sms, cudaStream_t stream);
// Sorts the keys of `ks` (all (k ^ ks.xr) - key_lo < key_range, distinct) into
// out (may alias the keys: every read precedes every write). ctrl->total =
// distinct keys, ctrl->bad_keys = keys out of range, ctrl->error != 0 on a
// protocol timeout (the state must then be re-initialised). `saved` holds
// G * S / 32 words when plan.P == 2.
cudaError_t launch_fused_sort(const KeySplit& ks, std::uint64_t key_range, std::uint32_t key_lo,
                              std::uint32_t* out, Ctrl* ctrl, void* state, std::uint32_t* saved,
                              const FusedPlan& plan, cudaStream_t stream,
                              unsigned long long* trace = nullptr, std::uint32_t* gbits = nullptr);
constexpr int KF_TRACE_WORDS = 15;  // per CTA: start, prod0, cons0, prod1, cons1, counts, end, spins x2,
                                    // producer thread 0 clocks: wait, rank, barrier A, scan, scatter, store

// KS (small.cu): a small sort in one cooperative launch — keys ORed into the
// cached global bitset, a grid barrier, per-CTA slices counted from registers,
// tagged count exchange, extraction straight from registers.
constexpr int KS_MAXG = 1024;    // CTAs (one per SM) the state is sized for
constexpr int KS_MAX_PER = 8;    // 16-byte bitset vectors per thread
struct SmallPlan {
    bool ok = false;
    int G = 0;                   // CTAs
    std::uint32_t per = 0;       // vectors per thread
    std::uint32_t total_v = 0;   // vectors covering the key range
};
struct SmallArgs {
    KeySplit ks;
    std::uint32_t lo;            // keys x with (x ^ xr) - lo > range_m1 are bad
    std::uint32_t range_m1;
    std::uint32_t* gbits;        // all-zero global bitset (>= total_v vectors); all-zero again afterwards
    std::uint32_t per, total_v;
    std::uint32_t* out;
    Ctrl* ctrl;                  // zeroed by CTA 0 before the barrier (no memset needed)
    unsigned long long* sync;    // monotonic arrival counter (G per launch)
    std::uint32_t* ghist;        // 2 x KS_MAXG: keys per owning slice, by launch parity (the other
                                 // parity's entries are zeroed for the next launch)
    std::uint32_t per_magic;     // ceil(2^32 / per): slice of key offset x = umulhi(x >> 17, per_magic)
    unsigned long long* trace;   // optional: KS_TRACE_WORDS globaltimer stamps per CTA
    int prefetch;                // prefetch the CTA's bitset slice into L2 before the REDs
};
constexpr int KS_TRACE_WORDS = 8;  // start, scattered, barrier passed, counted (offset known), -, end
SmallPlan plan_small(std::uint64_t key_range, int ctas);
std::size_t small_state_bytes();
cudaError_t configure_small(int device, LaunchGeometry* geo);
// state: small_state_bytes() bytes, zeroed once (and again after a fault).
cudaError_t launch_small_sort(const KeySplit& ks, std::uint64_t key_range, std::uint32_t key_lo,
                              std::uint32_t* out, Ctrl* ctrl, void* state,
                              const SmallPlan& plan, std::uint32_t* gbits, cudaStream_t stream,
                              unsigned long long* trace = nullptr, int prefetch = 1);

// K0: ctrl->max_key = max(keys) (only for sorts without a key-range hint).
cudaError_t launch_key_max(const std::uint32_t* keys, std::size_t n, Ctrl* ctrl,
                           const LaunchGeometry& geo, cudaStream_t stream, std::uint32_t xr = 0);

}  // namespace bws_gpu
